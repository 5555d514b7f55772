"""Single-GPU run of the p2p exchange kernels (n=1 self-exchange) so ncu can
profile k_reduce<EpiPush>, k_owner_apply and the stitch without peer waits."""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, '.')
from paper_1808_02621_b200 import ops
from paper_1808_02621_b200.model import VariableSpec, partition_bounds
from paper_1808_02621_b200.protocol import slab_layout
from paper_1808_02621_b200.runner import ShardedTable
from paper_1808_02621_b200.synth import TableShape, make_sparse_batch
from paper_1808_02621_b200.xchg import PeerExchange

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29650")
dist.init_process_group("gloo", rank=0, world_size=1)
from paper_1808_02621_b200 import _lib
for kv in filter(None, os.environ.get("HP_KNOBS", "").split(",")):  # A/B: NAME=INT
    k, v = kv.split("=")
    getattr(_lib.load(), f"hp_debug_set_{k}")(int(v))
dev = torch.device("cuda:0")
t = TableShape("softmax", 800_000, 512, 2560, sampled=8192)
P = 8
owner = np.zeros(P, np.int32)
bounds = partition_bounds(t.V, P)
_, base, rows = slab_layout(bounds, owner, 0)
cap = t.T + t.sampled
x = PeerExchange(1, 0, t.D, cap, rows, dev)
tab = ShardedTable(VariableSpec("softmax", t.V, 4 * t.D, 0.01, "sparse", True), P, owner, 0,
                   ops.OptimizerConfig("adagrad", lr=0.2), dev, seed=1, w_storage=lambda n: x.w[:n])
gb = torch.from_numpy(base).to(dev)
rng = np.random.default_rng(0)
ids, vals = make_sparse_batch(t, rng)
ids, vals = torch.from_numpy(ids).to(dev), torch.from_numpy(vals).to(dev)
out_b = {"send_ids": torch.empty(cap, dtype=torch.int64, device=dev),
         "inv": torch.empty(cap, dtype=torch.int32, device=dev),
         "dest_counts": torch.empty(1, dtype=torch.int32, device=dev),
         "n_uniq": torch.empty(1, dtype=torch.int32, device=dev)}
out = torch.empty(cap, t.D, device=dev)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
for s in range(steps):
    x.plan(ids, t.V, P, tab.owner_dev, gb, out_b, tab.ws)
    x.push_plan(vals, t.V, P, out_b, gb, tab.ws)
    x.merge_apply(tab.slab(), tab.optimizer.c_struct(s + 1, 1.0))
    x.stitch(out_b["inv"][:cap], out)
torch.cuda.synchronize()
if len(sys.argv) > 2 and sys.argv[2] == "time":  # per-phase CUDA-event times, GPU backlogged
    names = ["plan", "push", "apply", "stitch"]
    acc = {k: [] for k in names}
    for s in range(20):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        torch.cuda._sleep(20_000_000)
        ev[0].record()
        x.plan(ids, t.V, P, tab.owner_dev, gb, out_b, tab.ws); ev[1].record()
        x.push_plan(vals, t.V, P, out_b, gb, tab.ws); ev[2].record()
        x.merge_apply(tab.slab(), tab.optimizer.c_struct(s + 10, 1.0)); ev[3].record()
        x.stitch(out_b["inv"][:cap], out); ev[4].record()
        torch.cuda.synchronize()
        for i, k in enumerate(names):
            acc[k].append(ev[i].elapsed_time(ev[i + 1]) * 1e3)
    print({k: round(float(np.median(v)), 1) for k, v in acc.items()})
print("status", x.status(), "U", out_b["n_uniq"].item())
x.close()
