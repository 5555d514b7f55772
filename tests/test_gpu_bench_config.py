"""Parity of the EXACT benchmarked configuration (BASELINE configs[1], the
workload bench.py times at N=1): two 800k x 512 fp32 tables, T = 2560 and
2560 + 8192 sampled ids per step, 9.4M dense, Adagrad (lr 0.2, acc0 0.1),
P = 8, driven as bench.py drives it (one eager pipelined rotation, then CUDA
graphs of 2 steps each), against the C oracle (oracle/check.py)."""

import json

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("workload", ["lm1b", "nmt"])
def test_bench_config_bit_exact(cuda, workload):
    import paper_1808_02621_b200 as hp
    from oracle.check import check_runner_n1
    from paper_1808_02621_b200.synth import WORKLOADS, make_batch

    wl = WORKLOADS[workload]
    graph = hp.load_graph_spec(json.dumps(wl.graph_json()))
    cluster = hp.ClusterSpec.b200_box(1)
    plan = hp.transform_hybrid(graph, cluster, partitions={t.name: wl.partitions for t in wl.tables})
    runner = hp.HybridRunner(plan, graph, cluster, optimizer=hp.OptimizerConfig(**wl.optimizer),
                             device=cuda, seed=0)
    host = [make_batch(wl, seed=1 + i, rank=0) for i in range(6)]  # 3 plan slots: 2 ahead
    dev = [{k: ((torch.from_numpy(v[0]).to(cuda), torch.from_numpy(v[1]).to(cuda))
                if isinstance(v, tuple) else torch.from_numpy(v).to(cuda)) for k, v in b.items()}
           for b in host]
    out = check_runner_n1(runner, wl, host, dev, steps_per_graph=2, replays=1)
    assert runner.lookahead == 2
    assert out["steps"] == 12 and all(v > 1000 for v in out["rows"].values())
    runner.close()
