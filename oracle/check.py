"""End-to-end parity check of a single-GPU HybridRunner on ITS OWN benchmark
configuration (TEST INFRASTRUCTURE ONLY: used by tests/ and by
``bench.py --check`` before, never inside, the timed region).

The runner is driven exactly as bench.py drives it — one eager pipelined
rotation, then CUDA-graph replays of G steps per graph — and every step is
mirrored on the C oracle (oracle/hp_oracle.c, bit-identical to oracle.py) over
lazily paged full-size tables initialised at the touched rows. After the
replays the pulled rows of the last step, every touched table row and every
touched optimizer-state row must be bit-identical.
"""

from __future__ import annotations

import numpy as np

from . import coracle
from . import oracle as orc

F32 = np.float32


def _rows_of(tab, rows, torch, which=None):
    """Rows of a single-GPU ShardedTable (P partitions, all homed on rank 0)."""
    b = tab.bounds
    p = np.searchsorted(b, rows, side="right") - 1
    srow = tab.part_base_host[p] + rows - b[p]
    src = tab.w if which is None else tab.state[which]
    return src[torch.from_numpy(srow).to(src.device)].cpu().numpy()


def check_runner_n1(runner, wl, host_batches: list, dev_batches: list,
                    steps_per_graph: int = 2, replays: int = 2) -> dict:
    import torch

    if runner.world_size != 1:
        raise ValueError("check_runner_n1 is the single-GPU check")
    R = len(dev_batches)
    names = [v.name for v in runner.graph.variables]
    opt = runner.optimizer
    hpar = {"lr": opt.lr, "beta1": opt.beta1, "beta2": opt.beta2, "eps": opt.eps}
    states = {}
    for t in wl.tables:
        touched = np.concatenate([b[t.name][0] for b in host_batches])
        states[t.name] = orc.lazy_state(opt.kind, t.V, t.D, runner.seed * 1000 + names.index(t.name),
                                        touched, opt.init_acc)
    step = [0]
    last = {}

    def oracle_step(k):
        step[0] += 1
        for t in wl.tables:
            res = coracle.sparse_step(states[t.name], opt.kind, hpar, step[0],
                                      [host_batches[k][t.name]], t.V, 1, np.zeros(1, np.int32),
                                      aggregation=runner.aggregation)
            last[t.name] = res[0]["out"]

    # the bench's timed path: eager rotation (inside capture_pipelined), then graphs
    graphs = runner.capture_pipelined(dev_batches, steps_per_graph=steps_per_graph)
    for k in range(R):
        oracle_step(k)
    G = steps_per_graph
    for _ in range(replays):
        for g in range(R // G):
            graphs[g].replay()
            for j in range(G):
                oracle_step(g * G + j)
    torch.cuda.synchronize()
    runner.check_errors(sync=True)
    checked = {"steps": step[0], "rows": {}}
    for t in wl.tables:
        got = runner.outputs[t.name].cpu().numpy()
        if not np.array_equal(got, last[t.name]):
            bad = int((got != last[t.name]).any(axis=1).sum())
            raise AssertionError(f"{t.name}: pulled rows differ from the oracle ({bad} rows)")
        rows = np.unique(np.concatenate([b[t.name][0] for b in host_batches]))
        rows = rows[(rows >= 0) & (rows < t.V)]
        tab = runner.tables[t.name]
        if not np.array_equal(_rows_of(tab, rows, torch), states[t.name]["w"][rows]):
            raise AssertionError(f"{t.name}: updated table rows differ from the oracle")
        keys = {"adagrad": ["acc"], "adam": ["m", "v"]}.get(opt.kind, [])
        for i, key in enumerate(keys):
            if not np.array_equal(_rows_of(tab, rows, torch, i), states[t.name][key][rows]):
                raise AssertionError(f"{t.name}: optimizer state {key} differs from the oracle")
        checked["rows"][t.name] = int(rows.size)
    for name in wl.dense:
        k = (step[0] - 1) % R  # the dense mean at n = 1 is the last step's gradient itself
        ref = torch.from_numpy(host_batches[k][name]).to(runner.dense_dtype)
        if not torch.equal(runner.dense_out[name].reshape(-1).cpu(), ref):
            raise AssertionError(f"{name}: dense output differs")
    del graphs
    return checked
