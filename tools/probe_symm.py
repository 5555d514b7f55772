"""Does torch symmetric memory give a multicast (NVLS) pointer on this box?
torchrun --nproc-per-node N tools/probe_symm.py"""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

rank = int(os.environ["RANK"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
t = symm_mem.empty(1 << 20, dtype=torch.float32, device=f"cuda:{rank}")
h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
print(rank, "mc_ptr", hex(getattr(h, "multicast_ptr", 0) or 0), "buf_ptrs", [hex(p) for p in h.buffer_ptrs],
      "signal_pad", hex(h.signal_pad_ptrs[rank]) if hasattr(h, "signal_pad_ptrs") else None, flush=True)
dist.barrier()
dist.destroy_process_group()
