"""Device-timed partition-count search (Parallax's P search)
with the reference's own tune_evaluator; one rank per GPU.

python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
    --master-port 29620 tools/tune_p.py [workload] [iterations]
"""
import json, os, sys, time
import torch
import torch.distributed as dist
sys.path.insert(0, '.')
import paper_1808_02621_b200 as hp
from paper_1808_02621_b200.synth import WORKLOADS, make_batch

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "lm1b"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
comm = hp.Comm.from_torch_distributed()
graph = hp.load_graph_spec(json.dumps(wl.graph_json()))
cluster = hp.ClusterSpec.b200_box(world)


def mk(i):
    b = make_batch(wl, seed=100 + i, rank=rank)
    return {k: ((torch.from_numpy(v[0]).to(dev), torch.from_numpy(v[1]).to(dev))
                if isinstance(v, tuple) else torch.from_numpy(v).to(dev)) for k, v in b.items()}


log = []
ev = hp.device_evaluator(graph, cluster, mk, rank=rank, world_size=world, comm=comm,
                         optimizer=hp.OptimizerConfig(**wl.optimizer), iterations=iters, log=log)
cands = [v for v in graph.variables if v.kind == "sparse" and v.partitionable]
t0 = time.perf_counter()
res = hp.tune_evaluator(ev, start_p=min(cluster.machines, min(v.elements for v in cands)),
                        threshold=0.10, max_p=min(v.elements for v in cands))
wall = time.perf_counter() - t0
if rank == 0:
    out = res.to_dict() | {"n_gpus": world, "workload": wl.name, "iterations_per_sample": iters,
                           "search_wall_s": wall,
                           "words_per_s": {p: world * wl.words_per_worker / (t * 1e-6)
                                           for p, t in log}}
    print("TUNE " + json.dumps(out), flush=True)
comm.close()
dist.destroy_process_group()
