"""Raw NVLink peer store/load throughput between rank 0 and rank 1 (instrumentation)."""
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
S = 64 * 1024 * 1024  # 256 MB of fp32
d = DenseExchange(world, rank, S, torch.float32, dev)
lib = _lib.load()
res = {}
if rank == 0:
    st = torch.cuda.current_stream()
    for mode in (0, 1, 2, 3):
        for blocks in (74, 148, 296, 592, 1184):
            call("hp_debug_nvlink_bench", d.handle, 1, mode, blocks, st.cuda_stream)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                call("hp_debug_nvlink_bench", d.handle, 1, mode, blocks, st.cuda_stream)
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) * 1e3 / 5
            res[(mode, blocks)] = S * 4 / (us * 1e-6) / 1e9
    names = {0: "store x1", 1: "load x1", 2: "store x4", 3: "load x4"}
    for (m, bl), gbs in res.items():
        print(f"{names[m]:9s} blocks={bl:5d}  {gbs:7.1f} GB/s", flush=True)
dist.barrier()
d.close()
dist.destroy_process_group()
