"""Failure behaviour and API hygiene of the device path:

* ids outside [0, V) are DROPPED on the device exactly as the oracle drops
  them (no row updated, zero row pulled, inv = -1), never clamped onto a row;
* HybridRunner raises from the next step() when a device error bit was set,
  without synchronising the hot path;
* the dense K7 output never aliases or overwrites a caller's gradient tensor,
  and at n = 1 with fp32 and 'mean' nothing is launched for it.
"""

import json

import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu
F32 = np.float32


def _t(x, dev):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


def _with_bad(rng, ids, V, k):
    ids = ids.copy()
    bad = rng.choice(len(ids), k, replace=False)
    ids[bad[: k // 2]] = V + rng.integers(0, 1000, k // 2)
    ids[bad[k // 2:]] = -1 - rng.integers(0, 1000, k - k // 2)
    return ids


@pytest.mark.parametrize("T,V,D,P,n,k", [(3000, 50_000, 64, 8, 4, 40),       # cluster path
                                          (40_000, 300_000, 32, 8, 3, 500),   # multi-kernel path
                                          (20_000, 999, 8, 4, 2, 17),          # long dropped segment
                                          (3000, 100_000, 16, 4096, 8, 30)])   # P > cluster maximum
def test_k1_drops_out_of_range_ids(cuda, T, V, D, P, n, k):
    from paper_1808_02621_b200 import ops
    from paper_1808_02621_b200.synth import zipf_ids

    rng = np.random.default_rng(T + k)
    ids = _with_bad(rng, zipf_ids(rng, V, T), V, k)
    vals = rng.standard_normal((T, D), dtype=F32)
    owner = orc.owner_table("embedding", P, n)
    ref = orc.sort_dedup_route(ids, vals, V, P, owner, n)
    ws = ops.Workspace(cuda)
    got = ops.sort_dedup_route(_t(ids, cuda), _t(vals, cuda), V, P, _t(owner, cuda), n, ws)
    torch.cuda.synchronize()
    U = int(got["n_uniq"].item())
    assert U == ref["n_uniq"]
    assert ops.plan_status(ws) & 1
    assert np.array_equal(got["send_ids"][:U].cpu().numpy(), ref["send_ids"])
    assert np.array_equal(got["counts"][:U].cpu().numpy(), ref["counts"])
    assert np.array_equal(got["inv"][:T].cpu().numpy(), ref["inv"])
    assert np.array_equal(got["dest_counts"].cpu().numpy(), ref["dest_counts"])
    assert np.array_equal(got["send_rows"][:U].cpu().numpy(), ref["send_rows"])


def test_all_ids_out_of_range(cuda):
    from paper_1808_02621_b200 import ops

    ws = ops.Workspace(cuda)
    owner = _t(orc.owner_table("e", 4, 2), cuda)
    ids = torch.tensor([100, 101, -5, 100], dtype=torch.int64, device=cuda)
    got = ops.sort_dedup_route(ids, torch.ones(4, 8, device=cuda), 100, 4, owner, 2, ws)
    torch.cuda.synchronize()
    assert int(got["n_uniq"].item()) == 0
    assert got["dest_counts"].tolist() == [0, 0]
    assert got["inv"][:4].tolist() == [-1] * 4
    assert ops.plan_status(ws) == 1


@pytest.mark.parametrize("opt", ["sgd", "adagrad"])
def test_local_apply_and_gather_drop_bad_ids(cuda, opt):
    """n == 1 fused path (apply plan + K4 + K5) with bad ids == oracle.sparse_step."""
    from paper_1808_02621_b200 import ops
    from paper_1808_02621_b200.model import VariableSpec
    from paper_1808_02621_b200.runner import ShardedTable
    from paper_1808_02621_b200.synth import zipf_ids

    V, D, P, T = 100_000, 128, 4, 9000
    rng = np.random.default_rng(4)
    owner = np.zeros(P, dtype=np.int32)
    tab = ShardedTable(VariableSpec("t", V, 4 * D, 0.1, "sparse", True), P, owner, 0,
                       ops.OptimizerConfig(kind=opt, lr=0.1), cuda, seed=5)
    state = orc.init_state(opt, V, D, 5, 0.1)
    ids = _with_bad(rng, zipf_ids(rng, V, T), V, 64)
    vals = rng.standard_normal((T, D), dtype=F32)
    res = orc.sparse_step(state, opt, {"lr": 0.1}, 1, [(ids, vals)], V, P, owner)
    ops.local_apply(_t(ids, cuda), _t(vals, cuda), tab.slab(), tab.optimizer.c_struct(1, 1.0),
                    tab.ws)
    out = torch.empty(T, D, device=cuda)
    ops.gather_rows(tab.slab(), _t(ids, cuda), out)
    torch.cuda.synchronize()
    assert ops.plan_status(tab.ws) & 1
    assert np.array_equal(out.cpu().numpy(), res[0]["out"])
    assert np.array_equal(tab.w.cpu().numpy(), state["w"])


def _small_runner(cuda, dense_dtype=torch.float32, opt="adagrad"):
    import paper_1808_02621_b200 as hp
    from paper_1808_02621_b200.synth import TableShape, Workload

    wl = Workload("robust", [TableShape("embedding", 20_000, 64, 1000)], {"lstm": 4096},
                  {"kind": opt, "lr": 0.2, "init_acc": 0.1}, 1000)
    graph = hp.load_graph_spec(json.dumps(wl.graph_json()))
    cluster = hp.ClusterSpec.b200_box(1)
    plan = hp.transform_hybrid(graph, cluster)
    runner = hp.HybridRunner(plan, graph, cluster, optimizer=hp.OptimizerConfig(**wl.optimizer),
                             device=cuda, seed=1, dense_dtype=dense_dtype)
    return wl, runner


def _dev_batch(wl, cuda, seed, bad=0):
    from paper_1808_02621_b200.synth import make_batch

    b = make_batch(wl, seed=seed, rank=0)
    if bad:
        ids = b["embedding"][0].copy()
        ids[:bad] = wl.tables[0].V + np.arange(bad)
        b["embedding"] = (ids, b["embedding"][1])
    return b, {k: ((_t(v[0], cuda), _t(v[1], cuda)) if isinstance(v, tuple) else _t(v, cuda))
               for k, v in b.items()}


def test_runner_raises_after_a_bad_id(cuda):
    from paper_1808_02621_b200._lib import HybridPathError

    wl, runner = _small_runner(cuda)
    _, good = _dev_batch(wl, cuda, 1)
    _, bad = _dev_batch(wl, cuda, 2, bad=3)
    runner.step(good, timed=False)
    runner.step(good, timed=False)
    runner.check_errors(sync=True)  # clean so far
    runner.step(bad, timed=False)   # enqueued; the error is read one step later
    torch.cuda.synchronize()
    with pytest.raises(HybridPathError, match="outside"):
        runner.step(good, timed=False)
    runner.step(good, timed=False)  # words cleared after raising; good steps run on
    runner.check_errors(sync=True)
    runner.close()


def test_runner_raises_after_a_bad_id_in_graph_replays(cuda):
    from paper_1808_02621_b200._lib import HybridPathError

    wl, runner = _small_runner(cuda)
    dev = [_dev_batch(wl, cuda, s)[1] for s in (1, 2)]
    graphs = runner.capture_pipelined(dev)
    for _ in range(2):
        for g in graphs:
            g.replay()
    runner.check_errors(sync=True)
    dev[1]["embedding"][0][:2] = -7  # a bad id inside a captured batch
    for _ in range(2):
        for g in graphs:
            g.replay()
    with pytest.raises(HybridPathError, match="outside"):
        runner.check_errors(sync=True)
    runner.close()


@pytest.mark.parametrize("dense_dtype", [torch.float32, torch.bfloat16])
def test_dense_output_never_writes_caller_tensors(cuda, dense_dtype):
    """Round-1 bug: dense_out reused the caller's first gradient as the output
    buffer and later steps overwrote it. Caller tensors must stay bit-unchanged;
    at n = 1 with fp32 'mean' K7 launches nothing."""
    from paper_1808_02621_b200 import ops

    wl, runner = _small_runner(cuda, dense_dtype)
    host = [_dev_batch(wl, cuda, s) for s in (1, 2, 3)]
    keep = [h["lstm"].copy() for h, _ in host]
    for step, (h, d) in enumerate(host):
        runner.step(d, timed=False)
        torch.cuda.synchronize()
        ref = torch.from_numpy(h["lstm"]).to(dense_dtype)
        assert torch.equal(runner.dense_out["lstm"].cpu(), ref)
        for k in range(step + 1):  # every earlier caller tensor untouched
            assert np.array_equal(host[k][1]["lstm"].cpu().numpy(), keep[k])
    l0 = ops.launch_count()
    runner._dense(host[0][1])
    launched = ops.launch_count() - l0
    if dense_dtype == torch.float32:
        assert launched == 0 and runner.dense_out["lstm"] is host[0][1]["lstm"]
    else:
        assert launched == 1 and runner.dense_out["lstm"].data_ptr() != host[0][1]["lstm"].data_ptr()
    runner.close()
