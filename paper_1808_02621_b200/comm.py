"""Process-group plumbing: one NCCL communicator per process/GPU.

``torch.distributed`` (any backend) only carries the 128-byte NCCL unique id
from rank 0 to the others; all data movement goes through the library's own
communicator (``hp_comm_init``) on the caller's CUDA stream.
"""

from __future__ import annotations

import ctypes as C

import torch

from ._lib import call, load


class Comm:
    def __init__(self, handle: int, rank: int, world_size: int):
        self.handle = handle
        self.rank = rank
        self.world_size = world_size

    @property
    def ptr(self):
        return self.handle

    @classmethod
    def from_torch_distributed(cls, group=None) -> "Comm":
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        lib = load()
        nbytes = lib.hp_nccl_unique_id_bytes()
        uid = (C.c_ubyte * nbytes)()
        if rank == 0:
            call("hp_nccl_get_unique_id", C.addressof(uid))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        raw = (C.c_ubyte * nbytes).from_buffer_copy(box[0])
        handle = C.c_void_p()
        call("hp_comm_init", C.byref(handle), world, rank, C.addressof(raw))
        return cls(handle.value, rank, world)

    def alltoall_counts(self, send: torch.Tensor, recv: torch.Tensor) -> None:
        call("hp_alltoall_counts", self.handle, send.data_ptr(), recv.data_ptr(),
             torch.cuda.current_stream().cuda_stream)

    def push(self, send_ids, send_rows, send_counts, recv_ids, recv_rows, recv_counts, D) -> None:
        sc = (C.c_int32 * self.world_size)(*send_counts)
        rc = (C.c_int32 * self.world_size)(*recv_counts)
        call("hp_exchange_push", self.handle, send_ids.data_ptr(), send_rows.data_ptr(), sc,
             recv_ids.data_ptr(), recv_rows.data_ptr(), rc, D,
             torch.cuda.current_stream().cuda_stream)

    def pull(self, owner_rows, owner_counts, worker_rows, worker_counts, D) -> None:
        oc = (C.c_int32 * self.world_size)(*owner_counts)
        wc = (C.c_int32 * self.world_size)(*worker_counts)
        call("hp_exchange_pull", self.handle, owner_rows.data_ptr(), oc, worker_rows.data_ptr(),
             wc, D, torch.cuda.current_stream().cuda_stream)

    def status(self) -> int:
        """ncclCommGetAsyncError of the communicator (0 = success; host-only)."""
        r = C.c_int32(0)
        call("hp_comm_status", self.handle, C.addressof(r))
        return r.value

    def close(self) -> None:
        if self.handle:
            call("hp_comm_destroy", self.handle)
            self.handle = None
