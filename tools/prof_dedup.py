"""Per-phase clock64 profile of the cluster dedup kernel (instrumentation)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1808_02621_b200 import ops, _lib
from paper_1808_02621_b200.synth import zipf_ids, log_uniform_ids

dev = torch.device('cuda:0')
lib = _lib.load()
prof = torch.zeros(16 * 16, dtype=torch.int64, device=dev)
rng = np.random.default_rng(0)
import itertools
for nt, (T, V) in itertools.product((1024, 512, 256), ((2560, 800_000), (10752, 800_000), (2560, 37_000))):
    lib.hp_debug_set_cluster_threads(nt)
    ids = torch.from_numpy(zipf_ids(rng, V, T)).to(dev)
    ws = ops.Workspace(dev)
    for it in range(30):
        if it == 29:
            lib.hp_debug_set_profile(prof.data_ptr())
        ops.dedup_plan(ids, V, 8, torch.zeros(8, dtype=torch.int32, device=dev), 1, 512, ws)
        torch.cuda.synchronize()
    lib.hp_debug_set_profile(None)
    p = prof.view(16, 16).cpu().numpy()
    print(f"NT={nt} T={T} V={V}")
    for c in range(1):
        row = p[c]
        n = int((row != 0).sum())
        if n < 2:
            continue
        d = np.diff(row[:n])
        print(f"  cta{c}: total {row[n-1]-row[0]:7d} cyc  phases {[int(x) for x in d]}")
    prof.zero_()
