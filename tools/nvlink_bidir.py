"""NVLink peer-store/load throughput with every rank active at once (instrumentation).

Each rank streams S*4 bytes to (or from) rank (rank+1) % n with k_nvl_bench while
all other ranks do the same, so every GPU's NVLink carries traffic in both
directions; prints per-rank GB/s (one direction) per mode and grid size.
"""
import os, sys
import torch
import torch.distributed as dist
sys.path.insert(0, '.')
from paper_1808_02621_b200 import _lib
from paper_1808_02621_b200._lib import call
from paper_1808_02621_b200.xchg import DenseExchange

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
S = 16 * 1024 * 1024 * world  # chunk of 64 MB per rank
d = DenseExchange(world, rank, S, torch.float32, dev)
_lib.load()
peer = (rank + 1) % world
st = torch.cuda.current_stream()
names = {0: "store x1", 1: "load x1", 2: "store x4", 3: "load x4"}
res = []
for mode in (2, 3):
    for blocks in (148, 296, 592):
        call("hp_debug_nvlink_bench", d.handle, peer, mode, blocks, st.cuda_stream)
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            call("hp_debug_nvlink_bench", d.handle, peer, mode, blocks, st.cuda_stream)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / 5
        res.append((names[mode], blocks, round(S * 4 / (us * 1e-6) / 1e9, 1)))
out = [None] * world
dist.all_gather_object(out, res)
if rank == 0:
    for r, o in enumerate(out):
        print(f"rank {r}:", o, flush=True)
dist.barrier()
d.close()
dist.destroy_process_group()
