"""Device parity: every CUDA entry point against the CPU oracle on identical
seeded inputs. Integer/index outputs and gathered rows are compared
bit-exactly; summed rows and optimizer rows are ALSO bit-exact (same fp32
operation order as oracle.tree_sum / oracle.apply_*), which is stronger than
the north star's 1e-5 relative bar; the dense allreduce is compared within
1e-5 relative + 1e-6 absolute (NCCL's reduction order is not observable)."""

import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu
F32 = np.float32


def _t(x, dev):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


def _ids(rng, V, T, kind):
    if kind == "zipf":
        from paper_1808_02621_b200.synth import zipf_ids

        return zipf_ids(rng, V, T)
    if kind == "uniform":
        return rng.integers(0, V, T).astype(np.int64)
    if kind == "one":
        return np.full(T, V // 3, dtype=np.int64)
    if kind == "few":
        return rng.integers(0, 3, T).astype(np.int64) * (V // 3)
    raise ValueError(kind)


K1_CASES = [
    # (T, V, D, P, n, kind)
    (1, 10, 4, 1, 1, "uniform"),
    (7, 10, 4, 3, 2, "uniform"),
    (2560, 10_000, 128, 2, 2, "zipf"),
    (2560, 800_000, 512, 8, 8, "zipf"),
    (10752, 800_000, 512, 16, 8, "zipf"),
    (16384, 37_000, 1024, 8, 4, "zipf"),      # small-path maximum
    (16385, 37_000, 256, 8, 4, "zipf"),       # first large-path size
    (5000, 1000, 64, 5, 3, "one"),            # one segment of 5000 -> 2-level tree
    (20000, 999, 36, 4, 2, "few"),            # large path, 3 hot segments
    (200_000, 10_000_000, 128, 128, 8, "zipf"),
    (300_000, 1 << 20, 8, 33, 7, "uniform"),
    (3000, 100_000, 16, 4096, 8, "uniform"),   # P beyond the cluster path -> large path
    (2560, 800_000, 512, 2048, 8, "zipf"),     # cluster path, maximum P
    (4097, 65_536, 8, 3, 3, "zipf"),           # 3-CTA data in a 4-CTA cluster
    (8193, 1 << 24, 4, 2, 2, "uniform"),       # 3 radix passes, 8-CTA cluster
]


@pytest.fixture(params=[0, 1], ids=["k_reduce", "k_rowstream"])
def level0(request, cuda):
    """Run the test with each level-0 reduce kernel (hp_debug_set_rowstream)."""
    from paper_1808_02621_b200 import _lib

    lib = _lib.load()
    lib.hp_debug_set_rowstream(request.param)
    yield request.param
    lib.hp_debug_set_rowstream(0)


@pytest.mark.parametrize("T,V,D,P,n,kind", K1_CASES)
def test_sort_dedup_route_bit_exact(cuda, level0, T, V, D, P, n, kind):
    from paper_1808_02621_b200 import ops

    rng = np.random.default_rng(T + V + D)
    ids = _ids(rng, V, T, kind)
    vals = rng.standard_normal((T, D), dtype=F32)
    owner = orc.owner_table("embedding", P, n)
    ref = orc.sort_dedup_route(ids, vals, V, P, owner, n)
    ws = ops.Workspace(cuda)
    got = ops.sort_dedup_route(_t(ids, cuda), _t(vals, cuda), V, P, _t(owner, cuda), n, ws)
    torch.cuda.synchronize()
    U = int(got["n_uniq"].item())
    assert U == ref["n_uniq"]
    assert ops.plan_status(ws) == 0
    assert np.array_equal(got["send_ids"][:U].cpu().numpy(), ref["send_ids"])
    assert np.array_equal(got["counts"][:U].cpu().numpy(), ref["counts"])
    assert np.array_equal(got["inv"][:T].cpu().numpy(), ref["inv"])
    assert np.array_equal(got["dest_counts"].cpu().numpy(), ref["dest_counts"])
    assert np.array_equal(got["send_rows"][:U].cpu().numpy(), ref["send_rows"])


def test_sort_dedup_route_empty(cuda):
    from paper_1808_02621_b200 import ops

    ws = ops.Workspace(cuda)
    owner = _t(orc.owner_table("e", 4, 2), cuda)
    got = ops.sort_dedup_route(torch.zeros(0, dtype=torch.int64, device=cuda),
                               torch.zeros(0, 8, device=cuda), 100, 4, owner, 2, ws)
    torch.cuda.synchronize()
    assert int(got["n_uniq"].item()) == 0
    assert got["dest_counts"].tolist() == [0, 0]


def test_out_of_range_ids_flagged(cuda):
    from paper_1808_02621_b200 import ops

    ws = ops.Workspace(cuda)
    ids = torch.tensor([1, 5, 100, -1], dtype=torch.int64, device=cuda)
    ops.dedup_plan(ids, 10, 1, None, 1, 4, ws)
    assert ops.plan_status(ws) & 1


def _slab_for(V, D, P, owner, rank, opt, seed, dev, init_acc=0.1):
    """A ShardedTable-like slab for rank `rank` plus its oracle full table."""
    from paper_1808_02621_b200 import ops
    from paper_1808_02621_b200.model import VariableSpec
    from paper_1808_02621_b200.runner import ShardedTable

    tab = ShardedTable(VariableSpec("t", V, 4 * D, 0.1, "sparse", True), P, owner, rank,
                       ops.OptimizerConfig(kind=opt, lr=0.1, init_acc=init_acc), dev, seed=seed)
    state = orc.init_state(opt, V, D, seed, init_acc)
    return tab, state


def _gather_full(tab):
    """Reassemble the rows this rank homes into {global row: row}."""
    out = {}
    w = tab.w.cpu().numpy()
    for p in tab.owned:
        lo, hi = int(tab.bounds[p]), int(tab.bounds[p + 1])
        b = int(tab.part_base_host[p])
        out.update({r: w[b + r - lo] for r in range(lo, hi)})
    return out


@pytest.mark.parametrize("opt", ["sgd", "adagrad", "adam"])
@pytest.mark.parametrize("V,D,P,n,T", [(5000, 128, 6, 3, 3000), (800_000, 512, 8, 8, 2560),
                                       (37_000, 1024, 4, 2, 20000)])
def test_merge_apply_bit_exact(cuda, level0, opt, V, D, P, n, T):
    """Owner K4: rows received from n sources (in source order) merged + applied."""
    from paper_1808_02621_b200 import ops

    rng = np.random.default_rng(V + D)
    owner = orc.owner_table("t", P, n)
    rank = int(owner[0])
    tab, state = _slab_for(V, D, P, owner, rank, opt, seed=11, dev=cuda)
    hpar = {"lr": 0.1, "beta1": 0.9, "beta2": 0.999, "eps": 1e-8}
    mine = np.flatnonzero(owner == rank)
    b = orc.partition_bounds(V, P)
    got_ids, got_rows = [], []
    for s in range(n):
        parts = rng.choice(mine, size=len(mine))
        rows = np.unique(np.concatenate([rng.integers(b[p], b[p + 1], T // (n * len(mine)) + 1)
                                         for p in parts]))
        got_ids.append(rows)
        got_rows.append(rng.standard_normal((rows.size, D), dtype=F32))
    ids = np.concatenate(got_ids)
    rows = np.concatenate(got_rows)
    for step in (1, 2):
        scale = F32(1.0 / n)
        uniq, sums, _, _ = orc.grouped_tree_sum(ids, rows)
        orc.apply_rows(opt, state, uniq, sums * scale, hpar, step)
        o = tab.optimizer.c_struct(step, 1.0 / n)
        ops.merge_apply(_t(ids, cuda), _t(rows, cuda), ids.size, tab.slab(), o, tab.ws)
    torch.cuda.synchronize()
    assert ops.plan_status(tab.ws) == 0
    full = _gather_full(tab)
    rows_homed = np.array(sorted(full))
    assert np.array_equal(np.stack([full[r] for r in rows_homed]), state["w"][rows_homed])
    if opt != "sgd":
        s0 = tab.state[0].cpu().numpy()
        key = "acc" if opt == "adagrad" else "m"
        for p in tab.owned:
            lo, hi, base = int(b[p]), int(b[p + 1]), int(tab.part_base_host[p])
            assert np.array_equal(s0[base:base + hi - lo], state[key][lo:hi])


@pytest.mark.parametrize("opt", ["sgd", "adagrad", "adam"])
def test_local_apply_and_gather(cuda, level0, opt):
    """n == 1 fused step (K1+K4 then K5) == oracle.sparse_step with one worker."""
    from paper_1808_02621_b200 import ops
    from paper_1808_02621_b200.synth import zipf_ids

    V, D, P, T = 200_000, 256, 4, 12_000
    rng = np.random.default_rng(5)
    owner = np.zeros(P, dtype=np.int32)
    tab, state = _slab_for(V, D, P, owner, 0, opt, seed=3, dev=cuda)
    hpar = {"lr": 0.1, "beta1": 0.9, "beta2": 0.999, "eps": 1e-8}
    for step in (1, 2, 3):
        ids = zipf_ids(rng, V, T)
        vals = rng.standard_normal((T, D), dtype=F32)
        res = orc.sparse_step(state, opt, hpar, step, [(ids, vals)], V, P, owner)
        o = tab.optimizer.c_struct(step, 1.0)
        ops.local_apply(_t(ids, cuda), _t(vals, cuda), tab.slab(), o, tab.ws)
        out = torch.empty(T, D, device=cuda)
        ops.gather_rows(tab.slab(), _t(ids, cuda), out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), res[0]["out"])
    assert np.array_equal(tab.w.cpu().numpy(), state["w"])


@pytest.mark.parametrize("opt", ["adagrad", "adam"])
@pytest.mark.parametrize("mode", ["side", "side_b8", "side_tma", "side_cbcast", "side_lite",
                                  "one_stream", "build_order"])
def test_apply_plan_pull_split_bit_exact(cuda, opt, mode):
    """K4 + K5 fused (hp_apply_plan_pull) at the LM1B softmax shape: the short
    segments on a side stream beside the long chain (default; also with the
    8-rows-in-flight long-chunk reduce, and with the long roots + their pull in
    one work-queue kernel), on one stream, and with plans in build order
    (hp_debug_set_split_long(0)) == oracle."""
    from paper_1808_02621_b200 import _lib, ops
    from paper_1808_02621_b200.synth import log_uniform_ids, zipf_ids

    V, D, P, T = 800_000, 512, 8, 2560
    rng = np.random.default_rng(17)
    owner = np.zeros(P, dtype=np.int32)
    tab, state = _slab_for(V, D, P, owner, 0, opt, seed=5, dev=cuda)
    hpar = {"lr": 0.1, "beta1": 0.9, "beta2": 0.999, "eps": 1e-8}
    side = torch.cuda.Stream(device=cuda) if mode.startswith("side") else None
    _lib.load().hp_debug_set_split_long(0 if mode == "build_order" else 1)
    _lib.load().hp_debug_set_long_b8(1 if mode == "side_b8" else 0)
    _lib.load().hp_debug_set_cbcast(24 if mode == "side_cbcast" else 0)
    _lib.load().hp_debug_set_long_tma(2 if mode == "side_tma" else 0)
    _lib.load().hp_debug_set_comb_lite(1 if mode == "side_lite" else 0)
    try:
        for step in (1, 2):
            ids = np.concatenate([zipf_ids(rng, V, T), log_uniform_ids(rng, V, 8192)])
            ids[::997] = V + 5  # dropped ids: zero rows, no update
            vals = rng.standard_normal((ids.size, D), dtype=F32)
            res = orc.sparse_step(state, opt, hpar, step, [(ids, vals)], V, P, owner)
            o = tab.optimizer.c_struct(step, 1.0)
            ops.apply_plan_build(_t(ids, cuda), tab.slab(), tab.ws)
            out = torch.full((ids.size, D), float("nan"), device=cuda)
            ops.apply_plan_pull(_t(vals, cuda), ids.size, tab.slab(), o, out, tab.ws,
                                side_stream=side)
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy(), res[0]["out"]), step
        assert np.array_equal(tab.w.cpu().numpy(), state["w"])
    finally:
        _lib.load().hp_debug_set_split_long(1)
        _lib.load().hp_debug_set_long_b8(0)
        _lib.load().hp_debug_set_cbcast(0)
        _lib.load().hp_debug_set_long_tma(0)
        _lib.load().hp_debug_set_comb_lite(0)


def test_init_rows_bit_exact(cuda):
    from paper_1808_02621_b200 import ops

    w = torch.empty(300, 36, device=cuda)
    ops.init_rows(w, 1234, seed=77)
    assert np.array_equal(w.cpu().numpy(), orc.init_rows(1234, 1534, 36, 77))


def test_stitch_and_gather_exact(cuda):
    from paper_1808_02621_b200 import ops

    rng = np.random.default_rng(0)
    rows = rng.standard_normal((1000, 512), dtype=F32)
    inv = rng.integers(0, 1000, 7777).astype(np.int32)
    out = torch.empty(7777, 512, device=cuda)
    ops.stitch(_t(rows, cuda), _t(inv, cuda), out)
    assert np.array_equal(out.cpu().numpy(), rows[inv])


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16])
def test_dense_scale_cast_single_rank(cuda, dtype):
    from paper_1808_02621_b200 import ops

    rng = np.random.default_rng(1)
    g = rng.standard_normal(1_000_003, dtype=F32)
    gt = _t(g, cuda)
    out = torch.empty(g.size, dtype=dtype, device=cuda)
    ops.dense_allreduce_scale_cast(None, gt, out, 0.5)
    ref = torch.from_numpy(g * F32(0.5)).to(dtype)
    assert torch.equal(out.cpu(), ref)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16])
def test_dense_bf16_input_scale_cast(cuda, dtype):
    """K7 with bf16 gradients (in_dtype) at n = 1: exact widening, scale, cast;
    odd size (vector body + scalar tail)."""
    from paper_1808_02621_b200 import ops

    rng = np.random.default_rng(9)
    g16 = torch.from_numpy(rng.standard_normal(100_003, dtype=F32)).to(torch.bfloat16)
    out = torch.empty(g16.numel(), dtype=dtype, device=cuda)
    ops.dense_allreduce_scale_cast(None, g16.to(cuda), out, 0.25)
    ref = torch.from_numpy(g16.float().numpy() * F32(0.25)).to(dtype)
    assert torch.equal(out.cpu(), ref)


def test_runner_single_gpu_matches_oracle(cuda):
    """HybridRunner at n=1 on a reduced LM graph: pulled rows, tables and dense."""
    import paper_1808_02621_b200 as hp
    from paper_1808_02621_b200.synth import TableShape, Workload, make_batch

    wl = Workload("lm_small", [TableShape("embedding", 50_000, 128, 2560),
                               TableShape("softmax", 50_000, 128, 2560, sampled=2048)],
                  {"lstm": 100_000}, {"kind": "adagrad", "lr": 0.2, "init_acc": 0.1}, 2560)
    graph = hp.load_graph_spec(__import__("json").dumps(wl.graph_json()))
    cluster = hp.ClusterSpec.b200_box(1)
    plan = hp.transform_hybrid(graph, cluster, partitions={"embedding": 8, "softmax": 8})
    runner = hp.HybridRunner(plan, graph, cluster, optimizer=hp.OptimizerConfig(**wl.optimizer),
                             device=cuda, seed=2)
    states = {t.name: orc.init_state("adagrad", t.V, t.D, 2 * 1000 + i + 1, 0.1)
              for i, t in enumerate(wl.tables)}  # dense var is index 0
    for step in (1, 2):
        b = make_batch(wl, seed=step, rank=0)
        batch = {k: ((_t(v[0], cuda), _t(v[1], cuda)) if isinstance(v, tuple) else _t(v, cuda))
                 for k, v in b.items()}
        stats = runner.step(batch)
        assert stats.iter_time_us > 0
        for t in wl.tables:
            ids, vals = b[t.name]
            res = orc.sparse_step(states[t.name], "adagrad", {"lr": 0.2}, step, [(ids, vals)],
                                  t.V, 1, np.zeros(1, np.int32))
            assert np.array_equal(runner.outputs[t.name].cpu().numpy(), res[0]["out"])
        assert torch.equal(runner.dense_out["lstm"].cpu(), torch.from_numpy(b["lstm"]))
    for t in wl.tables:
        assert np.array_equal(runner.tables[t.name].w.cpu().numpy(), states[t.name]["w"])


@pytest.mark.parametrize("opt", ["adagrad", "adam"])
def test_runner_pipelined_and_graphs_match_oracle(cuda, opt):
    """Plans built one step ahead (next_batch) and the pipelined graph rotation
    give bit-identical tables and pulled rows (Adam: device step counter)."""
    import json

    import paper_1808_02621_b200 as hp
    from paper_1808_02621_b200.synth import TableShape, Workload, make_batch

    wl = Workload("pipe", [TableShape("embedding", 40_000, 128, 2560),
                           TableShape("softmax", 40_000, 256, 2560, sampled=3000)],
                  {"lstm": 10_000}, {"kind": opt, "lr": 0.2, "init_acc": 0.1}, 2560)
    graph = hp.load_graph_spec(json.dumps(wl.graph_json()))
    cluster = hp.ClusterSpec.b200_box(1)
    plan = hp.transform_hybrid(graph, cluster)
    runner = hp.HybridRunner(plan, graph, cluster, optimizer=hp.OptimizerConfig(**wl.optimizer),
                             device=cuda, seed=7)
    states = {t.name: orc.init_state(opt, t.V, t.D, 7 * 1000 + i + 1, 0.1)
              for i, t in enumerate(wl.tables)}
    hpar = {"lr": 0.2, "beta1": 0.9, "beta2": 0.999, "eps": 1e-8}
    step = [0]
    host = [make_batch(wl, seed=s, rank=0) for s in (1, 2)]
    dev = [{k: ((_t(v[0], cuda), _t(v[1], cuda)) if isinstance(v, tuple) else _t(v, cuda))
            for k, v in b.items()} for b in host]
    order = []

    def advance(r):
        step[0] += 1
        out = {}
        for t in wl.tables:
            ids, vals = host[r][t.name]
            out[t.name] = orc.sparse_step(states[t.name], opt, hpar, step[0], [(ids, vals)], t.V,
                                          1, np.zeros(1, np.int32))[0]["out"]
        return out

    def check(r):
        ref = advance(r)
        for t in wl.tables:
            assert np.array_equal(runner.outputs[t.name].cpu().numpy(), ref[t.name]), (r, t.name)

    runner.prefetch(dev[0])
    for r in (0, 1, 0):
        runner.step(dev[r], next_batch=dev[(r + 1) % 2])
        check(r)
    graphs = runner.capture_pipelined(dev)  # eagerly runs batch 0, 1 (rotation warm-up)
    torch.cuda.synchronize()
    for r in (0, 1):
        advance(r)
    for rep in range(2):
        for r in (0, 1):
            graphs[r].replay()
            torch.cuda.synchronize()
            check(r)
    # two steps per graph (the bench default), interleaved with the single-step graphs
    multi = runner.capture_pipelined(dev, steps_per_graph=2)  # eager warm-up: batch 0, 1
    torch.cuda.synchronize()
    for r in (0, 1):
        advance(r)
    for rep in range(2):
        multi[0].replay()
        torch.cuda.synchronize()
        advance(0)
        check(1)
    graphs[0].replay()
    torch.cuda.synchronize()
    check(0)
    graphs[1].replay()
    torch.cuda.synchronize()
    check(1)
    for t in wl.tables:
        assert np.array_equal(runner.tables[t.name].w.cpu().numpy(), states[t.name]["w"])
