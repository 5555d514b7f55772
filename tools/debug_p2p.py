"""2-rank smoke of the peer-memory exchange with signal-word dumps."""
import os, sys, time
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, '.')
from paper_1808_02621_b200 import ops
from paper_1808_02621_b200.xchg import PeerExchange
from paper_1808_02621_b200.runner import ShardedTable
from paper_1808_02621_b200.model import VariableSpec, partition_bounds
from paper_1808_02621_b200.protocol import slab_layout
from oracle import oracle as orc

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
V, D, P, T = 1000, 8, 4, 64
owner = orc.owner_table("t", P, world)
bounds = partition_bounds(V, P)
_, _, rows = slab_layout(bounds, owner, rank)
x = PeerExchange(world, rank, D, T, max(rows, 1), dev)
print(rank, "window ok", x.debug_sig(), flush=True)
tab = ShardedTable(VariableSpec("t", V, 4 * D, 0.1, "sparse", True), P, owner, rank,
                   ops.OptimizerConfig("sgd", lr=0.1), dev, seed=1, w_storage=lambda n: x.w[:n])
gb = np.zeros(P, np.int64)
for r in range(world):
    _, base, _ = slab_layout(bounds, owner, r)
    gb[base >= 0] = base[base >= 0]
gb = torch.from_numpy(gb).to(dev)
rng = np.random.default_rng(rank)
ids = torch.from_numpy(rng.integers(0, V, T)).to(dev)
vals = torch.randn(T, D, device=dev)
r = ops.sort_dedup_route(ids, vals, V, P, tab.owner_dev, world, tab.ws)
torch.cuda.synchronize()
print(rank, "dest_counts", r["dest_counts"].tolist(), "U", r["n_uniq"].item(), flush=True)
x.push(r["send_ids"], r["send_rows"], r["dest_counts"], T)
torch.cuda.synchronize()
print(rank, "after push", x.debug_sig(), flush=True)
dist.barrier()
print(rank, "after barrier", x.debug_sig(), flush=True)
x.merge_apply(tab.slab(), ops.OptimizerConfig("sgd", lr=0.1).c_struct(1, 0.5))
torch.cuda.synchronize()
print(rank, "after apply", x.debug_sig(), flush=True)
pulled = torch.empty(T, D, device=dev)
x.pull(r["send_ids"], r["n_uniq"], T, tab.owner_dev, gb, V, P, pulled)
torch.cuda.synchronize()
print(rank, "after pull", x.debug_sig(), "status", x.status(), flush=True)
x.close()
dist.destroy_process_group()
