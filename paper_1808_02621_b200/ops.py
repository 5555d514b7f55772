"""Typed PyTorch wrappers over the C ABI (one call = one C entry point).

Every function checks dtype / device / contiguity, marshals ``data_ptr()`` and
the current CUDA stream, and raises :class:`HybridPathError` on a non-zero
return. No op has a CPU path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import Optim, Slab, call, load


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _p(t):
    return None if t is None else t.data_ptr()


def _need(t: torch.Tensor, dtype, name: str, dim: int | None = None) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dim is not None and t.dim() != dim:
        raise ValueError(f"{name} must be {dim}-D, got shape {tuple(t.shape)}")


class Workspace:
    """Grow-only device scratch buffer shared by consecutive calls on one stream."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.buf = torch.empty(0, dtype=torch.uint8, device=self.device)

    def get(self, nbytes: int) -> torch.Tensor:
        if self.buf.numel() < nbytes:
            self.buf = torch.empty(int(nbytes * 1.25) + 4096, dtype=torch.uint8, device=self.device)
            self.buf[:256].zero_()  # the plan counters (incl. the error word) start clean
        return self.buf

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()

    @property
    def nbytes(self) -> int:
        return self.buf.numel()


class ErrorWords:
    """Pinned, device-mapped host words that device error bits are collected into
    (``hp_err_collect``): reading them never synchronises the GPU."""

    def __init__(self, n: int):
        h, d = C.c_void_p(), C.c_void_p()
        call("hp_err_host_alloc", n, C.byref(h), C.byref(d))
        self.n, self._host, self._dev = n, h.value, d.value
        self.words = (C.c_int32 * n).from_address(self._host)

    def collect(self, slot: int, sources, stream=None) -> None:
        """OR ``(device word pointer, shift)`` sources into host word ``slot``."""
        sources = [(p, sh) for p, sh in sources if p]
        if not sources:
            return
        ptrs = (C.c_void_p * len(sources))(*[p for p, _ in sources])
        shifts = (C.c_int32 * len(sources))(*[sh for _, sh in sources])
        call("hp_err_collect", ptrs, shifts, len(sources), self._dev + 4 * slot, _stream(stream))

    def read(self) -> list:
        return [int(self.words[i]) for i in range(self.n)]

    def clear(self) -> None:
        for i in range(self.n):
            self.words[i] = 0

    def close(self) -> None:
        if self._host:
            call("hp_err_host_free", self._host)
            self._host = None


class StepGraph:
    """A CUDA graph captured with torch (``torch.cuda.CUDAGraph(keep_graph=True)``,
    so torch's private memory pool and stream bookkeeping apply) and
    instantiated by the library with per-node priorities
    (``hp_graph_instantiate``): each kernel node keeps the priority of the
    stream it was captured on, so the plan streams' dedup is dispatched ahead
    of the tables' reduce instead of after it drains. ``node_priority=False``
    instantiates without the flag (A/B). ``replay()`` launches on the current stream."""

    def __init__(self, node_priority: bool = True):
        import os

        # HP_STEPGRAPH=0 (default): torch instantiates and replays (measured:
        # launching through the library's own runtime made every replay ~15 us
        # slower, r2m); 1: library instantiate with node priorities; 2: torch
        # instantiate, library launch; F > 2: raw instantiate flags F (A/B)
        self.mode = int(os.environ.get("HP_STEPGRAPH", "0"))
        self.torch_replay = self.mode == 0
        self.graph = torch.cuda.CUDAGraph(keep_graph=not self.torch_replay)
        self.node_priority = node_priority
        self._exec = None
        self._owned = True

    def capture(self):
        return torch.cuda.graph(self.graph)

    def _instantiate(self) -> None:
        if self.mode == 2:
            self.graph.instantiate()
            self._exec, self._owned = self.graph.raw_cuda_graph_exec(), False
            return
        ex = C.c_void_p()
        flags = self.mode if self.mode > 2 else int(self.node_priority)
        call("hp_graph_instantiate", self.graph.raw_cuda_graph(), flags, C.byref(ex))
        self._exec = ex.value

    def replay(self) -> None:
        if self.torch_replay:
            self.graph.replay()
            return
        if self._exec is None:
            self._instantiate()
        call("hp_graph_launch", self._exec, _stream())

    def __del__(self):
        if getattr(self, "_exec", None) and getattr(self, "_owned", False):
            try:
                load().hp_graph_destroy(self._exec)
            except Exception:  # interpreter teardown
                pass
            self._exec = None


def plan_err_ptr(ws: "Workspace") -> int | None:
    """Device address of the error word of the plan in ``ws`` (None if unsized)."""
    if ws.nbytes == 0:
        return None
    out = C.c_void_p()
    call("hp_plan_err_ptr", ws.ptr, C.byref(out))
    return out.value


def dedup_ws_bytes(T: int, D: int, P: int, nranks: int = 1) -> int:
    return int(load().hp_dedup_ws_bytes(T, D, P, nranks))


@dataclass
class OptimizerConfig:
    """Sparse row optimizer: sgd | adagrad | adam."""

    kind: str = "adagrad"
    lr: float = 0.2
    init_acc: float = 0.1
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    def __post_init__(self):
        if self.kind not in _lib.HP_OPT:
            raise ValueError(f"unknown optimizer {self.kind!r}")

    def lr_t(self, step) -> np.ndarray:
        """Adam bias-corrected step size, float64 on the host, rounded to fp32."""
        step = np.asarray(step, dtype=np.float64)
        return (self.lr * np.sqrt(1.0 - self.beta2 ** step) / (1.0 - self.beta1 ** step)).astype(
            np.float32)

    def c_struct(self, step: int, agg_scale: float, lr_t_table=None, step_ctr=None) -> Optim:
        """Kernel parameters for one step. With ``lr_t_table`` (device float32,
        index = step) and ``step_ctr`` (device int32) Adam reads its step size
        on the device, so a captured graph stays correct across replays."""
        lr_t = float(self.lr_t(step)) if self.kind == "adam" else 0.0
        o = Optim(_lib.HP_OPT[self.kind], self.lr, self.beta1, self.beta2, 1.0 - self.beta1,
                  1.0 - self.beta2, self.eps, lr_t, agg_scale)
        if lr_t_table is not None:
            o.lr_t_table = lr_t_table.data_ptr()
            o.step_ctr = step_ctr.data_ptr()
            o.table_len = lr_t_table.numel()
        return o

    @property
    def n_state(self) -> int:
        return {"sgd": 0, "adagrad": 1, "adam": 2}[self.kind]


def sort_dedup_route(ids: torch.Tensor, vals: torch.Tensor, V: int, P: int, owner: torch.Tensor,
                     nranks: int, ws: Workspace, out: dict | None = None, stream=None) -> dict:
    """K1+K2: dedup + route one worker's IndexedSlices into send order."""
    _need(ids, torch.int64, "ids", 1)
    _need(vals, torch.float32, "vals", 2)
    _need(owner, torch.int32, "owner", 1)
    T, D = vals.shape
    if ids.numel() != T:
        raise ValueError("ids and vals disagree on T")
    dev = ids.device
    o = out if out is not None else {}
    if "send_rows" in o and (o["send_rows"].shape[0] < max(T, 1) or o["send_rows"].shape[1] != D
                             or o["dest_counts"].numel() != nranks):
        o.clear()
    o.setdefault("send_ids", torch.empty(max(T, 1), dtype=torch.int64, device=dev))
    o.setdefault("send_rows", torch.empty(max(T, 1), D, dtype=torch.float32, device=dev))
    o.setdefault("counts", torch.empty(max(T, 1), dtype=torch.int32, device=dev))
    o.setdefault("inv", torch.empty(max(T, 1), dtype=torch.int32, device=dev))
    o.setdefault("dest_counts", torch.empty(nranks, dtype=torch.int32, device=dev))
    o.setdefault("n_uniq", torch.empty(1, dtype=torch.int32, device=dev))
    need = dedup_ws_bytes(T, D, P, nranks)
    ws.get(need)
    call("hp_sort_dedup_route", _p(ids), _p(vals), T, D, V, P, _p(owner), nranks,
         _p(o["send_ids"]), _p(o["send_rows"]), _p(o["counts"]), _p(o["inv"]),
         _p(o["dest_counts"]), _p(o["n_uniq"]), ws.ptr, ws.nbytes, _stream(stream))
    return o


def dedup_plan(ids: torch.Tensor, V: int, P: int, owner: torch.Tensor | None, nranks: int, D: int,
               ws: Workspace, outputs: bool = True, stream=None) -> dict:
    """Index-only K1+K2 (no rows): send ids, counts, inverse map, dest counts.

    With ``outputs=False`` only the plan in ``ws`` is built (for apply_plan)."""
    _need(ids, torch.int64, "ids", 1)
    T = ids.numel()
    dev = ids.device
    if outputs:
        o = {"send_ids": torch.empty(max(T, 1), dtype=torch.int64, device=dev),
             "counts": torch.empty(max(T, 1), dtype=torch.int32, device=dev),
             "inv": torch.empty(max(T, 1), dtype=torch.int32, device=dev),
             "dest_counts": torch.empty(nranks, dtype=torch.int32, device=dev),
             "n_uniq": torch.empty(1, dtype=torch.int32, device=dev)}
    else:
        o = {k: None for k in ("send_ids", "counts", "inv", "dest_counts", "n_uniq")}
    ws.get(dedup_ws_bytes(T, D, P, nranks))
    call("hp_dedup_plan", _p(ids), T, D, V, P, _p(owner), nranks, _p(o["send_ids"]),
         _p(o["counts"]), _p(o["inv"]), _p(o["dest_counts"]), _p(o["n_uniq"]), ws.ptr, ws.nbytes,
         _stream(stream))
    return o


def plan_status(ws: Workspace, stream=None) -> int:
    err = C.c_int32(0)
    call("hp_plan_status", ws.ptr, C.addressof(err), _stream(stream))
    return err.value


def merge_apply(ids: torch.Tensor, rows: torch.Tensor, n: int, slab: Slab, opt: Optim,
                ws: Workspace, stream=None) -> None:
    """K4: merge received (id, row) pairs and apply the optimizer on the owner slab."""
    _need(ids, torch.int64, "ids", 1)
    _need(rows, torch.float32, "rows", 2)
    ws.get(dedup_ws_bytes(n, slab.D, slab.P))
    call("hp_merge_apply", _p(ids), _p(rows), n, slab, opt, ws.ptr, ws.nbytes, _stream(stream))


def local_apply(ids: torch.Tensor, vals: torch.Tensor, slab: Slab, opt: Optim, ws: Workspace,
                stream=None) -> None:
    """n == 1 fused K1+K4: dedup the worker's slices and apply straight to the slab."""
    _need(ids, torch.int64, "ids", 1)
    _need(vals, torch.float32, "vals", 2)
    T = ids.numel()
    ws.get(dedup_ws_bytes(T, slab.D, slab.P))
    call("hp_local_apply", _p(ids), _p(vals), T, slab, opt, ws.ptr, ws.nbytes, _stream(stream))


def apply_plan_build(ids: torch.Tensor, slab: Slab, ws: Workspace, n: int | None = None,
                     stream=None) -> None:
    """Index half of K4: dedup ids into a plan whose destinations are slab rows."""
    _need(ids, torch.int64, "ids", 1)
    n = ids.numel() if n is None else n
    ws.get(dedup_ws_bytes(n, slab.D, slab.P))
    call("hp_apply_plan_build", _p(ids), n, slab, ws.ptr, ws.nbytes, _stream(stream))


def apply_plan(rows: torch.Tensor, n: int, slab: Slab, opt: Optim, ws: Workspace,
               stream=None) -> None:
    """K4 only: reduce + apply with the plan apply_plan_build left in ``ws``."""
    _need(rows, torch.float32, "rows", 2)
    call("hp_apply_plan", _p(rows), n, slab, opt, ws.ptr, ws.nbytes, _stream(stream))


def apply_plan_pull(rows: torch.Tensor, n: int, slab: Slab, opt: Optim, out: torch.Tensor,
                    ws: Workspace, stream=None, side_stream=None) -> torch.Tensor:
    """K4 + K5 fused (n = 1): reduce + apply with the plan in ``ws`` and
    out[t] = the updated row of position t's id (``hp_apply_plan_pull``).
    ``side_stream``: the short segments run there, beside the long ones' chain."""
    _need(rows, torch.float32, "rows", 2)
    _need(out, torch.float32, "out", 2)
    if out.shape[0] < n or out.shape[1] != slab.D:
        raise ValueError(f"out must be at least [{n}, {slab.D}]")
    call("hp_apply_plan_pull", _p(rows), n, slab, opt, _p(out), ws.ptr, ws.nbytes, _stream(stream),
         None if side_stream is None else _stream(side_stream))
    return out


def step_counter_inc(ctr: torch.Tensor, stream=None) -> None:
    """++ctr on the device (the Adam step of graph-captured steps)."""
    call("hp_step_counter_inc", _p(ctr), _stream(stream))


def launch_count() -> int:
    """Kernels this library has launched so far in the process."""
    return int(load().hp_launch_count())


def gather_rows(slab: Slab, ids: torch.Tensor, out: torch.Tensor, n: int | None = None,
                n_dev: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """K5: out[i] = row ids[i] of this rank's slab."""
    _need(ids, torch.int64, "ids", 1)
    _need(out, torch.float32, "out", 2)
    n = ids.numel() if n is None else n
    call("hp_gather_rows", slab, _p(ids), n, _p(n_dev), _p(out), _stream(stream))
    return out


def plan_stitch(ws: Workspace, T: int, D: int, V: int, P: int, rows_ptr: int,
                out: torch.Tensor, stream=None) -> torch.Tensor:
    """K5 / K6 from the dedup plan in ``ws``: out[t] = rows[plan destination of
    position t] (slab rows of an apply plan / return rows of a send plan),
    TMA-broadcast once per unique row (``hp_plan_stitch``)."""
    _need(out, torch.float32, "out", 2)
    if out.shape[0] < T or out.shape[1] != D:
        raise ValueError(f"out must be at least [{T}, {D}]")
    call("hp_plan_stitch", ws.ptr, ws.nbytes, T, D, V, P, rows_ptr, _p(out), _stream(stream))
    return out


def stitch(rows: torch.Tensor, inv: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    """K6: out[t] = rows[inv[t]]."""
    _need(rows, torch.float32, "rows", 2)
    _need(inv, torch.int32, "inv", 1)
    _need(out, torch.float32, "out", 2)
    T, D = out.shape
    call("hp_stitch", _p(rows), _p(inv), T, D, _p(out), _stream(stream))
    return out


def init_rows(w: torch.Tensor, row_lo: int, seed: int, scale: float = 0.05, stream=None) -> None:
    _need(w, torch.float32, "w", 2)
    call("hp_init_rows", _p(w), row_lo, w.shape[0], w.shape[1], seed, scale, _stream(stream))


def fill(x: torch.Tensor, value: float, stream=None) -> None:
    _need(x, torch.float32, "x")
    call("hp_fill", _p(x), x.numel(), value, _stream(stream))


def dense_allreduce_scale_cast(comm, grad: torch.Tensor, out: torch.Tensor, scale: float,
                               stream=None, scratch: torch.Tensor | None = None) -> torch.Tensor:
    """K7: out = cast(scale * sum over ranks of grad). fp32 grad: reduced in
    place; bf16 grad (``hp_dense_allreduce_scale_cast_ex``): widened exactly to
    fp32 (into ``scratch``, fp32 of grad's size, when there is more than one rank)."""
    if grad.dtype not in (torch.float32, torch.bfloat16):
        raise TypeError("grad must be float32 or bfloat16")
    _need(grad, grad.dtype, "grad")
    if out.dtype not in (torch.float32, torch.bfloat16, torch.float16) or not out.is_contiguous():
        raise TypeError("out must be a contiguous float32/bfloat16/float16 tensor")
    if out.numel() != grad.numel():
        raise ValueError("grad and out sizes differ")
    code = _lib.HP_DTYPE[str(out.dtype).split(".")[1]]
    if grad.dtype == torch.float32:
        call("hp_dense_allreduce_scale_cast", comm, _p(grad), _p(out), grad.numel(), code, scale,
             _stream(stream))
        return out
    if scratch is not None:
        _need(scratch, torch.float32, "scratch")
        if scratch.numel() < grad.numel():
            raise ValueError("scratch must hold grad.numel() fp32 elements")
    call("hp_dense_allreduce_scale_cast_ex", comm, _p(grad), _lib.HP_DTYPE["bfloat16"], _p(out),
         grad.numel(), code, scale, None if scratch is None else _p(scratch), _stream(stream))
    return out


def allgather(comm, src: torch.Tensor, dst: torch.Tensor, stream=None) -> torch.Tensor:
    """AR for a sparse Weight: dst = concat over ranks of src (rank order)."""
    if not (src.is_contiguous() and dst.is_contiguous()) or src.dtype != dst.dtype:
        raise TypeError("src and dst must be contiguous tensors of one dtype")
    nb = src.numel() * src.element_size()
    if dst.numel() * dst.element_size() < nb * _lib.load().hp_comm_size(comm):
        raise ValueError("dst too small for the allgather")
    call("hp_allgather", comm, _p(src), _p(dst), nb, _stream(stream))
    return dst


def dense_reduce_bcast(comm, grad: torch.Tensor, out: torch.Tensor, scale: float, root: int,
                       stream=None) -> torch.Tensor:
    """PS for a dense Weight: out = cast(scale * sum over ranks of grad), reduced at ``root``."""
    _need(grad, torch.float32, "grad")
    if out.numel() != grad.numel() or not out.is_contiguous():
        raise ValueError("out must be contiguous with grad's size")
    code = _lib.HP_DTYPE[str(out.dtype).split(".")[1]]
    call("hp_dense_reduce_bcast", comm, _p(grad), _p(out), grad.numel(), code, scale, root,
         _stream(stream))
    return out
