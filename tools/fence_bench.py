"""Cost of the per-block publication fence vs grid size (instrumentation).

Rank 0 launches k_fence_bench (every block: optional peer stores, then a fence
variant + one atomic) for several grid sizes; prints us per launch."""
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
S = 16 * 1024 * 1024
d = DenseExchange(world, rank, S, torch.float32, dev)
_lib.load()
if rank == 0:
    st = torch.cuda.current_stream()
    names = {0: "none", 1: "fence.sc.sys", 2: "fence.sc.gpu", 3: "fence.acq_rel.sys"}
    for per_block in (0, 1024):
        for mode in (0, 1, 2, 3):
            row = []
            for blocks in (32, 148, 444, 1184):
                call("hp_debug_fence_bench", d.handle, 1, mode, blocks, per_block, st.cuda_stream)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(20):
                    call("hp_debug_fence_bench", d.handle, 1, mode, blocks, per_block, st.cuda_stream)
                b.record()
                torch.cuda.synchronize()
                row.append(round(a.elapsed_time(b) * 1e3 / 20, 2))
            print(f"per_block={per_block:5d} {names[mode]:18s} blocks 32/148/444/1184: {row} us", flush=True)
dist.barrier()
d.close()
dist.destroy_process_group()
