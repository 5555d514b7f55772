"""Multi-GPU kernel timeline from in-kernel globaltimer spans (instrumentation).

python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
    --master-port 29610 tools/span_multi.py [table|dense|lm1b] [pipelined]
Prints, per rank, each kernel type's [start, end] in us relative to the step's
first kernel (median over iterations).
"""
import json, os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, '.')
import paper_1808_02621_b200 as hp
from paper_1808_02621_b200 import _lib
from paper_1808_02621_b200.synth import WORKLOADS, TableShape, Workload, make_batch

NAMES = ["dedup", "reduce", "combine", "wait_push", "scatter", "apply", "wait_applied", "copy",
         "ar_scatter", "ar_wait0", "ar_rg", "ar_wait1", "publish", "applied", "reduce_short"]
which = sys.argv[1] if len(sys.argv) > 1 else "table"
pipelined = len(sys.argv) > 2 and sys.argv[2] in ("pipelined", "graph")
use_graph = len(sys.argv) > 2 and sys.argv[2] == "graph"  # replay the bench's pipelined graphs
if which == "table":
    wl = Workload("t", [TableShape("softmax", 800_000, 512, 2560, sampled=8192)], {},
                  {"kind": "adagrad", "lr": 0.2, "init_acc": 0.1}, 2560)
elif which == "table_emb":
    wl = Workload("t", [TableShape("embedding", 800_000, 512, 2560)], {},
                  {"kind": "adagrad", "lr": 0.2, "init_acc": 0.1}, 2560)
elif which == "dense":
    wl = Workload("d", [], {"lstm": 9_400_000}, {"kind": "adagrad", "lr": 0.2}, 2560)
else:
    wl = WORKLOADS[which]
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
comm = hp.Comm.from_torch_distributed()
graph = hp.load_graph_spec(json.dumps(wl.graph_json()))
cluster = hp.ClusterSpec.b200_box(world)
plan = hp.transform_hybrid(graph, cluster, partitions={t.name: 8 for t in wl.tables})
for kv in filter(None, os.environ.get("HP_KNOBS", "").split(",")):  # before the first plan
    k, v = kv.split("=")
    getattr(_lib.load(), f"hp_debug_set_{k}")(int(v))
runner = hp.HybridRunner(plan, graph, cluster, rank=rank, world_size=world, comm=comm,
                         optimizer=hp.OptimizerConfig(**wl.optimizer), device=dev)
bs = []
for s in (1, 2):
    b = make_batch(wl, seed=s, rank=rank)
    bs.append({k: ((torch.from_numpy(v[0]).to(dev), torch.from_numpy(v[1]).to(dev))
                   if isinstance(v, tuple) else torch.from_numpy(v).to(dev)) for k, v in b.items()})
lib = _lib.load()
for kv in filter(None, os.environ.get("HP_KNOBS", "").split(",")):  # A/B switches
    k, v = kv.split("=")
    getattr(lib, f"hp_debug_set_{k}")(int(v))
span = torch.zeros(32, dtype=torch.int64, device=dev)
graphs = None
if use_graph:
    graphs = runner.capture_pipelined(bs)
    for i in range(4):
        graphs[i % 2].replay()
elif pipelined:
    runner.prefetch(bs[0])
for i in range(0 if use_graph else 4):
    runner.step(bs[i % 2], timed=False, next_batch=bs[(i + 1) % 2] if pipelined else None)
torch.cuda.synchronize()
rows = []
for it in range(8):
    span.view(16, 2)[:, 0] = -1  # ~0 as unsigned
    span.view(16, 2)[:, 1] = 0
    lib.hp_debug_set_spans(span.data_ptr())
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda._sleep(20_000_000)
    if graphs:
        graphs[it % 2].replay()
    else:
        runner.step(bs[it % 2], timed=False, next_batch=bs[(it + 1) % 2] if pipelined else None)
    torch.cuda.synchronize()
    lib.hp_debug_set_spans(None)
    v = span.view(16, 2).cpu().numpy().astype(np.uint64)
    rows.append(v)
t0s = []
res = {}
for v in rows:
    valid = [(i, v[i, 0], v[i, 1]) for i in range(len(NAMES)) if v[i, 1] > 0]
    t0 = min(s for _, s, _ in valid)
    for i, s, e in valid:
        res.setdefault(NAMES[i], []).append(((s - t0) / 1e3, (e - t0) / 1e3))
summ = {k: (round(float(np.median([a for a, _ in x])), 1), round(float(np.median([b for _, b in x])), 1))
        for k, x in res.items()}
out = [None] * world
dist.all_gather_object(out, {"rank": rank, "spans_us": dict(sorted(summ.items(), key=lambda kv: kv[1][0]))})
if rank == 0:
    for o in out:
        print(json.dumps(o))
del graphs
torch.cuda.synchronize()
runner.close()
comm.close()
dist.destroy_process_group()
