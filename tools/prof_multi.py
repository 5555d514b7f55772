"""Per-phase device times of the multi-GPU step (CUDA events, GPU backlogged).

python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
    --master-port 29600 tools/prof_multi.py [workload] [exchange]
"""
import json, os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, '.')
import paper_1808_02621_b200 as hp
from paper_1808_02621_b200.synth import WORKLOADS, make_batch

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "lm1b"]
xmode = sys.argv[2] if len(sys.argv) > 2 else "p2p"
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
comm = hp.Comm.from_torch_distributed()
graph = hp.load_graph_spec(json.dumps(wl.graph_json()))
cluster = hp.ClusterSpec.b200_box(world)
plan = hp.transform_hybrid(graph, cluster, partitions={t.name: wl.partitions for t in wl.tables})
runner = hp.HybridRunner(plan, graph, cluster, rank=rank, world_size=world, comm=comm,
                         optimizer=hp.OptimizerConfig(**wl.optimizer), device=dev, exchange=xmode)
b = make_batch(wl, seed=1, rank=rank)
batch = {k: ((torch.from_numpy(v[0]).to(dev), torch.from_numpy(v[1]).to(dev))
             if isinstance(v, tuple) else torch.from_numpy(v).to(dev)) for k, v in b.items()}
b2 = make_batch(wl, seed=2, rank=rank)
batch2 = {k: ((torch.from_numpy(v[0]).to(dev), torch.from_numpy(v[1]).to(dev))
              if isinstance(v, tuple) else torch.from_numpy(v).to(dev)) for k, v in b2.items()}
for _ in range(3):
    runner.step(batch, timed=False)
torch.cuda.synchronize()
runner.kernel_events = {}
runner.concurrent_tables = os.environ.get("HP_PROF_CONCURRENT", "0") == "1"
for i in range(10):
    torch.cuda._sleep(50_000_000)
    dist.barrier()
    runner.step(batch, timed=False)
torch.cuda.synchronize()
res = {}
for key, evs in runner.kernel_events.items():
    d = [a.elapsed_time(c) * 1e3 for a, c in zip(evs[0::2], evs[1::2])]
    res[key] = round(float(np.median(d)), 1)
runner.concurrent_tables = True
for _ in range(3):
    runner.step(batch, timed=False)
stats = runner.step(batch, timed=True)
out = [None] * world
dist.all_gather_object(out, {"rank": rank, "us": res, "phases": stats.phase_times,
                             "iter_us": stats.iter_time_us,
                             "bytes": stats.per_machine_bytes.per_machine[rank]})
if rank == 0:
    for o in out:
        print(json.dumps(o))
runner.kernel_events = None
torch.cuda.synchronize()
runner.close()
comm.close()
dist.destroy_process_group()
