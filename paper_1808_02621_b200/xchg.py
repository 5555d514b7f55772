"""Python side of the NVLink peer-memory exchange (``hp_xchg_*`` in the C ABI).

One :class:`PeerExchange` per sparse table per rank: it owns the rank's
symmetric window (the table slab + inboxes + flags), swaps cudaIpc handles
with the other ranks over ``torch.distributed`` (plumbing only) and exposes
the three device-initiated phases push / merge_apply / pull.
"""

from __future__ import annotations

import ctypes as C

import torch

from ._lib import call, load


class _DevPtr:
    """Zero-copy tensor view of library-owned device memory."""

    def __init__(self, ptr: int, shape, typestr: str = "<f4"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def _connect(x, prefix: str, ipc, group, world) -> None:
    """Map the other ranks' windows: by cudaIpc handle (one process per GPU), or
    by address through ``world`` (n emulated ranks in one process). Peers
    address each other's windows with their own offsets, so the window shape
    (``x.shape``) must be identical on every rank: checked here."""
    if world is not None:
        world.register(x.KIND, x.rank, x)
        return
    import torch.distributed as dist

    handles = [None] * x.n
    dist.all_gather_object(handles, (bytes(ipc), x.shape), group=group)
    shapes = {h[1] for h in handles}
    if len(shapes) != 1:
        raise ValueError(f"{prefix}: window shapes differ across ranks: {sorted(shapes)}")
    for r, (h, _) in enumerate(handles):
        if r != x.rank:
            buf = (C.c_ubyte * 64).from_buffer_copy(h)
            call(f"{prefix}_open_peer", x.handle, r, C.addressof(buf))


class PeerExchange:
    """``world``: a :class:`~paper_1808_02621_b200.emulate.LocalWorld` links the
    windows of n emulated ranks of THIS process by address (one-GPU parity
    tests); otherwise cudaIpc handles are swapped over ``torch.distributed``."""

    KIND = "xchg"

    def __init__(self, n: int, rank: int, D: int, cap: int, rows_cap: int, device, group=None,
                 world=None):
        load()
        self.n, self.rank, self.D, self.cap = n, rank, D, cap
        self.shape = (n, D, cap, rows_cap)
        self.handle = C.c_void_p()
        ipc = (C.c_ubyte * 64)()
        wptr = C.c_void_p()
        call("hp_xchg_create", C.byref(self.handle), n, rank, D, cap, rows_cap, C.addressof(ipc),
             C.byref(wptr))
        self.w = torch.as_tensor(_DevPtr(wptr.value, (rows_cap, D)), device=device)
        _connect(self, "hp_xchg", ipc, group, world)

    def window_ptr(self) -> int:
        out = C.c_void_p()
        call("hp_xchg_window_ptr", self.handle, C.byref(out))
        return out.value

    def pull(self, ids, V: int, P: int, owner, glob_base, out) -> None:
        """out[t] = the current row of ids[t], read from its owner's slab (NVLink)."""
        call("hp_xchg_pull", self.handle, ids.data_ptr(), ids.numel(), V, P, owner.data_ptr(),
             glob_base.data_ptr(), out.data_ptr(), torch.cuda.current_stream().cuda_stream)

    @property
    def ret_ptr(self) -> int:
        """Device address of the returned rows [cap][D] (by send slot)."""
        out = C.c_void_p()
        call("hp_xchg_ret_ptr", self.handle, C.byref(out))
        return out.value

    def link_peer(self, rank: int, window: int) -> None:
        call("hp_xchg_set_peer_ptr", self.handle, rank, window)

    def push(self, ids, vals, V: int, P: int, owner, glob_base, out: dict, ws) -> dict:
        """Fused dedup + route + NVLink push; fills out[send_ids, inv, dest_counts, n_uniq]."""
        from .ops import dedup_ws_bytes

        T = ids.numel()
        ws.get(dedup_ws_bytes(T, self.D, P, self.n))
        call("hp_xchg_push", self.handle, ids.data_ptr(), vals.data_ptr(), T, V, P,
             owner.data_ptr(), glob_base.data_ptr(), out["send_ids"].data_ptr(),
             out["inv"].data_ptr(),
             out["dest_counts"].data_ptr(), out["n_uniq"].data_ptr(), ws.ptr, ws.nbytes,
             torch.cuda.current_stream().cuda_stream)
        return out

    def plan(self, ids, V: int, P: int, owner, glob_base, out: dict, ws) -> dict:
        """Index half of push: dedup + route into a send plan in ``ws`` (plus each
        send slot's destination: owner inbox index and slab row, from ``glob_base``)."""
        from .ops import dedup_ws_bytes

        T = ids.numel()
        ws.get(dedup_ws_bytes(T, self.D, P, self.n))
        call("hp_xchg_plan", self.handle, ids.data_ptr(), T, V, P, owner.data_ptr(),
             glob_base.data_ptr(), out["send_ids"].data_ptr(), out["inv"].data_ptr(), out["dest_counts"].data_ptr(),
             out["n_uniq"].data_ptr(), ws.ptr, ws.nbytes, torch.cuda.current_stream().cuda_stream)
        return out

    def push_plan(self, vals, V: int, P: int, out: dict, glob_base, ws, side_stream=None) -> None:
        """Value half of push: reduce with the plan in ``ws`` and store into owners'
        inboxes (``side_stream``: the short segments there, beside the long ones)."""
        call("hp_xchg_push_plan", self.handle, vals.data_ptr(), vals.shape[0], V, P,
             out["send_ids"].data_ptr(), out["dest_counts"].data_ptr(), glob_base.data_ptr(),
             ws.ptr, ws.nbytes, torch.cuda.current_stream().cuda_stream,
             None if side_stream is None else side_stream.cuda_stream)

    def wait(self, which: int) -> None:
        """0: until every source pushed; 1: until every owner applied."""
        call("hp_xchg_wait", self.handle, which, torch.cuda.current_stream().cuda_stream)

    def merge_apply(self, slab, opt, wait: bool = True) -> None:
        call("hp_xchg_merge_apply", self.handle, slab, opt, int(wait),
             torch.cuda.current_stream().cuda_stream)

    def stitch(self, inv, out, wait: bool = True) -> None:
        call("hp_xchg_stitch", self.handle, inv.data_ptr(), out.shape[0], out.data_ptr(),
             int(wait), torch.cuda.current_stream().cuda_stream)

    def stitch_plan(self, ws, T: int, V: int, P: int, out, wait: bool = True) -> None:
        """K6 through the send plan in ``ws``: out[t] = returned row of t's slot
        (the wait for every owner's apply folded into the kernel)."""
        call("hp_xchg_stitch_plan", self.handle, ws.ptr, ws.nbytes, T, V, P, out.data_ptr(),
             int(wait), torch.cuda.current_stream().cuda_stream)

    def recv_counts(self, out) -> None:
        call("hp_xchg_recv_counts", self.handle, out.data_ptr(),
             torch.cuda.current_stream().cuda_stream)

    def debug_sig(self) -> dict:
        buf = (C.c_int32 * 320)()
        call("hp_xchg_debug_sig", self.handle, C.addressof(buf),
             torch.cuda.current_stream().cuda_stream)
        v = list(buf)
        return {"push_flag": v[:self.n], "push_count": v[64:64 + self.n],
                "applied_flag": v[128:128 + self.n], "epoch": v[192], "err": v[193],
                "done": v[196:200], "push_off": v[256:256 + self.n]}

    def err_ptr(self) -> int:
        out = C.c_void_p()
        call("hp_xchg_err_ptr", self.handle, C.byref(out))
        return out.value

    def status(self) -> int:
        err = C.c_int32(0)
        call("hp_xchg_status", self.handle, C.addressof(err), torch.cuda.current_stream().cuda_stream)
        return err.value

    def close(self) -> None:
        if self.handle:
            torch.cuda.synchronize()
            call("hp_xchg_destroy", self.handle)
            self.handle = None


class DenseExchange:
    """K7 over peer memory for one dense Weight: a symmetric window holding the
    reduce slots and the output; ``allreduce(grad, scale)`` leaves
    cast(scale * sum_r grad_r) (summed in rank order) in ``self.out`` on every rank."""

    MODES = {"sm": 0, "ce": 1, "pipe": 2, "pull": 3}  # HP_DAR_* (include/hybridpath.h)
    KIND = "dar"

    def __init__(self, n: int, rank: int, numel: int, out_dtype, device, group=None,
                 mode: str = "ce", world=None, in_dtype=torch.float32):
        from ._lib import HP_DTYPE

        if numel % 4:
            raise ValueError("dense gradient size must be a multiple of 4")
        self.n, self.rank, self.numel = n, rank, numel
        self.handle = C.c_void_p()
        ipc = (C.c_ubyte * 64)()
        optr = C.c_void_p()
        code = HP_DTYPE[str(out_dtype).split(".")[1]]
        self.shape = (n, numel, code)
        call("hp_dar_create", C.byref(self.handle), n, rank, numel, code, C.addressof(ipc),
             C.byref(optr))
        _connect(self, "hp_dar", ipc, group, world)
        call("hp_dar_set_mode", self.handle, self.MODES[mode])
        if in_dtype not in (torch.float32, torch.bfloat16):
            raise TypeError("dense exchange input: float32 | bfloat16")
        if in_dtype == torch.bfloat16 and mode != "sm":
            raise ValueError("bf16 dense gradients need the SM-store exchange (mode 'sm')")
        self.in_dtype = in_dtype
        call("hp_dar_set_in_dtype", self.handle, HP_DTYPE[str(in_dtype).split(".")[1]])
        typestr = "<f4" if code == 0 else "<u2"
        t = torch.as_tensor(_DevPtr(optr.value, (numel,), typestr), device=device)
        self.out = t if code == 0 else t.view(torch.bfloat16)

    def window_ptr(self) -> int:
        out = C.c_void_p()
        call("hp_dar_window_ptr", self.handle, C.byref(out))
        return out.value

    def link_peer(self, rank: int, window: int) -> None:
        call("hp_dar_set_peer_ptr", self.handle, rank, window)

    def set_split(self, weights) -> None:
        """Share of the reduction per rank (hp_dar_set_split); identical on every rank."""
        w = (C.c_double * self.n)(*[float(x) for x in weights])
        call("hp_dar_set_split", self.handle, C.addressof(w))

    def allreduce(self, grad, scale: float) -> torch.Tensor:
        from .ops import _need

        _need(grad, self.in_dtype, "grad")
        if grad.numel() != self.numel:
            raise ValueError(f"grad has {grad.numel()} elements, the exchange was built for "
                             f"{self.numel}")
        call("hp_dar_allreduce", self.handle, grad.data_ptr(), scale,
             torch.cuda.current_stream().cuda_stream)
        return self.out

    def err_ptr(self) -> int:
        out = C.c_void_p()
        call("hp_dar_err_ptr", self.handle, C.byref(out))
        return out.value

    def status(self) -> int:
        err = C.c_int32(0)
        call("hp_dar_status", self.handle, C.addressof(err), torch.cuda.current_stream().cuda_stream)
        return err.value

    def close(self) -> None:
        if self.handle:
            torch.cuda.synchronize()
            call("hp_dar_destroy", self.handle)
            self.handle = None


class NvlsExchange:
    """K7 through the NVSwitch: the gradient is copied into a symmetric buffer
    bound to a multicast object (torch symmetric memory: allocation and
    rendezvous only); ``hp_nvls_allreduce`` reduces it in the switch
    (multimem.ld_reduce) and multicasts cast(scale * sum) into every rank's
    output (multimem.st). Same interface as :class:`DenseExchange`."""

    def __init__(self, n: int, rank: int, numel: int, out_dtype, device, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        from ._lib import HP_DTYPE, HybridPathError

        if numel % 4:
            raise ValueError("dense gradient size must be a multiple of 4")
        self.n, self.rank, self.numel = n, rank, numel
        self.S = -(-numel // (4 * n)) * 4 * n
        self.code = HP_DTYPE[str(out_dtype).split(".")[1]]
        if self.code not in (0, 1):
            raise ValueError("NVLS dense exchange: out dtype float32 | bfloat16")
        name = (group or dist.group.WORLD).group_name
        self.inp = symm_mem.empty(self.S, dtype=torch.float32, device=device)
        self.inp.zero_()
        self.outbuf = symm_mem.empty(self.S, dtype=out_dtype, device=device)
        hi = symm_mem.rendezvous(self.inp, name)
        ho = symm_mem.rendezvous(self.outbuf, name)
        self._handles = (hi, ho)
        if not hi.multicast_ptr or not ho.multicast_ptr:
            raise HybridPathError("NVLS multicast is not available on this system")
        self.mc_in, self.mc_out = hi.multicast_ptr, ho.multicast_ptr
        self.pads = torch.tensor(list(hi.signal_pad_ptrs), dtype=torch.int64, device=device)
        self.state = torch.zeros(2, dtype=torch.int32, device=device)
        torch.cuda.synchronize(device)
        dist.barrier(group=group)
        self.out = self.outbuf[:numel]

    def allreduce(self, grad, scale: float) -> torch.Tensor:
        if grad.dtype != torch.float32 or grad.numel() != self.numel or not grad.is_cuda:
            raise ValueError(f"grad must be a CUDA float32 tensor of {self.numel} elements")
        self.inp[:self.numel].copy_(grad.reshape(-1))
        call("hp_nvls_allreduce", self.mc_in, self.mc_out, self.S, self.n, self.rank, self.code,
             scale, self.pads.data_ptr(), self.state.data_ptr(),
             torch.cuda.current_stream().cuda_stream)
        return self.out

    def err_ptr(self) -> int:
        return self.state.data_ptr() + 4  # {epoch, error bits}

    def status(self) -> int:
        return int(self.state[1].item())

    def close(self) -> None:
        torch.cuda.synchronize()
        self._handles = None
