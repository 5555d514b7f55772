"""Diagnose the one-GPU emulated multi-rank exchange (tests/test_gpu_emulated.py):
one step per case, wall time, error bits and signal words per rank."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import paper_1808_02621_b200 as hp  # noqa: E402
from paper_1808_02621_b200.emulate import LocalWorld  # noqa: E402
from paper_1808_02621_b200.synth import TableShape, Workload, make_batch  # noqa: E402


def case(n, dex, opt, reserve=True, steps=2):
    dev = torch.device("cuda:0")
    wl = Workload("emu", [TableShape("embedding", 60_000, 128, 2560)], {"lstm": 100_000},
                  {"kind": opt, "lr": 0.2, "init_acc": 0.1}, 2560)
    graph = hp.load_graph_spec(json.dumps(wl.graph_json()))
    cl = hp.ClusterSpec.b200_box(n)
    plan = hp.transform_hybrid(graph, cl, partitions={"embedding": 8})
    world = LocalWorld(n)
    runs = [hp.HybridRunner(plan, graph, cl, rank=r, world_size=n, comm=world.comm(r),
                            optimizer=hp.OptimizerConfig(kind=opt, lr=0.2), device=dev, seed=3,
                            dense_exchange=dex) for r in range(n)]
    streams = [torch.cuda.Stream() for _ in range(n)]
    batches = []
    for r in range(n):
        b = make_batch(wl, 1, r)
        batches.append({k: ((torch.from_numpy(v[0]).to(dev), torch.from_numpy(v[1]).to(dev))
                            if isinstance(v, tuple) else torch.from_numpy(v).to(dev))
                        for k, v in b.items()})
    torch.cuda.synchronize()
    for st in range(steps):
        if reserve:
            for run, b in zip(runs, batches):
                run.reserve(b)
        t0 = time.time()
        for run, s, b in zip(runs, streams, batches):
            with torch.cuda.stream(s):
                run.step(b, timed=False)
        t1 = time.time()
        torch.cuda.synchronize()
        t2 = time.time()
        st_ = [run.exchange_status() for run in runs]
        sig = [run.xchg["embedding"].debug_sig() for run in runs]
        print(json.dumps({"case": [n, dex, opt, reserve], "step": st, "enqueue_s": round(t1 - t0, 4),
                          "sync_s": round(t2 - t1, 4), "status": st_,
                          "epochs": [s_["epoch"] for s_ in sig],
                          "push_flag": [s_["push_flag"] for s_ in sig],
                          "applied": [s_["applied_flag"] for s_ in sig]}), flush=True)
    for run in runs:
        run.close()


if __name__ == "__main__":
    which = sys.argv[1]
    if which == "basic":
        case(2, "p2p-sm", "adagrad", reserve=False)
        case(2, "p2p-sm", "adagrad", reserve=True)
    elif which == "ce":
        case(3, "p2p", "sgd", reserve=True)
    elif which == "pipe":
        from paper_1808_02621_b200 import _lib
        _lib.load().hp_debug_set_dar_blocks(24)
        case(2, "p2p-pipe", "adam", reserve=True)
