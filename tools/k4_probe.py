"""K4 (reduce + apply) in isolation on one GPU, per id distribution.

    python tools/k4_probe.py [--reps 30]

Prints µs per launch pair (k_reduce + k_combine) with L2 flushed between
launches, the algorithmic bytes and the fraction of MEASURED_PEAKS HBM.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1808_02621_b200 import ops  # noqa: E402
from paper_1808_02621_b200._lib import Slab  # noqa: E402
from paper_1808_02621_b200.synth import log_uniform_ids, zipf_ids  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--V", type=int, default=800_000)
    ap.add_argument("--D", type=int, default=512)
    ap.add_argument("--T", type=int, default=10752)
    ap.add_argument("--rowstream", type=int, default=1)
    ap.add_argument("--pdl", type=int, default=1)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    from paper_1808_02621_b200 import _lib
    lib = _lib.load()
    lib.hp_debug_set_rowstream(a.rowstream)
    lib.hp_debug_set_pdl(a.pdl)
    V, D, T = a.V, a.D, a.T
    w = torch.zeros(V, D, device=dev)
    acc = torch.full((V, D), 0.1, device=dev)
    pb = torch.tensor([0], dtype=torch.int64, device=dev)
    slab = Slab(w.data_ptr(), acc.data_ptr(), 0, pb.data_ptr(), V, 1, D)
    cfg = ops.OptimizerConfig("adagrad", lr=0.1)
    opt = cfg.c_struct(1, 1.0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    rng = np.random.default_rng(0)
    dists = {
        "distinct": rng.permutation(V)[:T],
        "pairs": np.repeat(rng.permutation(V)[:T // 2], 2),
        "chunk16": np.repeat(rng.permutation(V)[:T // 16], 16),
        "lm1b_softmax": np.concatenate([zipf_ids(rng, V, 2560), log_uniform_ids(rng, V, T - 2560)]),
        "lm1b_embedding": zipf_ids(rng, V, 2560),
        "one_hot_id": np.zeros(T, np.int64),
    }
    peak = 6434.2
    try:
        peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
    except Exception:
        pass
    for name, ids_np in dists.items():
        ids = torch.from_numpy(ids_np.astype(np.int64)).to(dev)
        n = ids.numel()
        vals = torch.randn(n, D, device=dev)
        ws = ops.Workspace(dev)
        ops.apply_plan_build(ids, slab, ws)
        torch.cuda.synchronize()
        U = len(np.unique(ids_np))
        ts = []
        for r in range(a.reps + 3):
            flush.fill_(r & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(1_000_000)
            e0.record()
            ops.apply_plan(vals, n, slab, opt, ws)
            e1.record()
            torch.cuda.synchronize()
            if r >= 3:
                ts.append(e0.elapsed_time(e1) * 1e3)
        us = float(np.median(ts))
        span = torch.zeros(32, dtype=torch.int64, device=dev)
        span[0::2] = (1 << 63) - 1
        lib.hp_debug_set_spans(span.data_ptr())
        flush.fill_(1)
        torch.cuda._sleep(1_000_000)
        ops.apply_plan(vals, n, slab, opt, ws)
        torch.cuda.synchronize()
        lib.hp_debug_set_spans(None)
        sp = span.cpu().numpy()
        t0 = sp[0::2].min()
        spans = {k: [round((sp[2 * i] - t0) / 1e3, 1), round((sp[2 * i + 1] - t0) / 1e3, 1)]
                 for i, k in [(1, "reduce"), (2, "combine")] if sp[2 * i + 1] > 0}
        algo = n * (4 + 4 * D) + U * (4 + 4 * D * 2 * 2)
        _, c = np.unique(ids_np, return_counts=True)
        print(json.dumps({"rowstream": a.rowstream, "pdl": a.pdl, "dist": name, "T": n, "U": U, "max_mult": int(c.max()), "us": round(us, 2),
                          "min_us": round(min(ts), 2), "GBps": round(algo / us / 1e3, 1),
                          "frac": round(algo / us / 1e3 / peak, 3), "spans": spans}), flush=True)


if __name__ == "__main__":
    main()
