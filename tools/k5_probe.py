"""K5 (the pull) in isolation: the plan-based TMA broadcast (hp_plan_stitch,
k_bcast_rows) vs the id-routed row copy (hp_gather_rows, k_copy_rows), per id
distribution and size, with L2 flushed before each launch.

    python tools/k5_probe.py [--reps 20]
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
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--D", type=int, default=512)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    V, D = 800_000, a.D
    w = torch.randn(V, D, device=dev)
    pb = torch.tensor([0], dtype=torch.int64, device=dev)
    slab = Slab(w.data_ptr(), None, None, pb.data_ptr(), V, 1, D)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6540.8
    rng = np.random.default_rng(0)
    cases = {
        "emb_2560": zipf_ids(rng, V, 2560),
        "softmax_10752": np.concatenate([zipf_ids(rng, V, 2560), log_uniform_ids(rng, V, 8192)]),
        "distinct_10752": rng.permutation(V)[:10752],
        "zipf_100k": zipf_ids(rng, V, 100_000),
        "distinct_200k": rng.permutation(V)[:200_000],
    }
    for name, ids_np in cases.items():
        ids = torch.from_numpy(ids_np.astype(np.int64)).to(dev)
        T = ids.numel()
        ws = ops.Workspace(dev)
        ops.apply_plan_build(ids, slab, ws)
        U = int(np.unique(ids_np).size)
        out = torch.empty(T, D, device=dev)
        ref = w[ids]
        res = {}
        from paper_1808_02621_b200 import _lib
        for kind in ("bcast", "bcast_reg", "copy"):
            _lib.load().hp_debug_set_bcast_tma(0 if kind == "bcast_reg" else 1)
            ts = []
            for r in range(a.reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(2_000_000)
                e0.record()
                if kind.startswith("bcast"):
                    ops.plan_stitch(ws, T, D, V, 1, w.data_ptr(), out)
                else:
                    ops.gather_rows(slab, ids, out)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            assert torch.equal(out, ref), kind
            us = float(np.median(ts))
            algo = T * 4 + U * 4 * D + T * 4 * D
            res[kind] = {"us": round(us, 2), "frac": round(algo / (us * 1e-6) / 1e9 / peak, 3)}
        print(json.dumps({"case": name, "T": T, "U": U, **res}), flush=True)


if __name__ == "__main__":
    main()
