"""CPU checks of the oracle itself (no GPU): it is the checker for every
device parity test, so its semantics are pinned here against float64
restatements and the planner's routing."""

import numpy as np
import pytest

import paper_1808_02621_b200 as hp
from oracle import oracle as orc

F32 = np.float32


def test_tree_sum_short_is_sequential():
    rng = np.random.default_rng(0)
    for L in (1, 2, 17, orc.CHUNK):
        x = rng.standard_normal((L, 8), dtype=F32)
        acc = np.zeros(8, F32)
        for r in x:
            acc = acc + r
        assert np.array_equal(orc.tree_sum(x), acc)


@pytest.mark.parametrize("L", [129, 1000, 16384, 40000])
def test_tree_sum_long_accuracy(L):
    rng = np.random.default_rng(L)
    x = rng.standard_normal((L, 16), dtype=F32)
    got = orc.tree_sum(x).astype(np.float64)
    ref = x.astype(np.float64).sum(0)
    scale = np.abs(x).astype(np.float64).sum(0)
    assert np.all(np.abs(got - ref) <= 1e-6 * scale)  # ~eps * depth * chunk bound
    # explicit two-level structure for L <= CHUNK^2
    if L <= orc.CHUNK ** 2:
        parts = [orc.seq_sum(x[i:i + orc.CHUNK]) for i in range(0, L, orc.CHUNK)]
        assert np.array_equal(got.astype(F32), orc.seq_sum(np.stack(parts)))


def test_sort_dedup_route_invariants():
    rng = np.random.default_rng(1)
    V, P, n, T, D = 5000, 7, 3, 3000, 8
    ids = rng.integers(0, V, T) ** 2 % V  # skewed
    vals = rng.standard_normal((T, D), dtype=F32)
    owner = orc.owner_table("embedding", P, n)
    r = orc.sort_dedup_route(ids, vals, V, P, owner, n)
    U = r["n_uniq"]
    assert U == len(np.unique(ids)) and r["counts"].sum() == T
    dest = owner[orc.partition_of(r["send_ids"], V, P)]
    key = dest.astype(np.int64) * V + r["send_ids"]
    assert np.all(np.diff(key) > 0)  # strictly ascending (owner, id)
    assert np.array_equal(np.bincount(dest, minlength=n), r["dest_counts"])
    assert np.array_equal(r["send_ids"][r["inv"]], ids)
    ref = np.zeros((U, D))
    np.add.at(ref, r["inv"], vals.astype(np.float64))
    assert np.allclose(r["send_rows"], ref, rtol=1e-5, atol=1e-5)


def test_empty_and_single():
    owner = orc.owner_table("e", 2, 2)
    r = orc.sort_dedup_route(np.zeros(0, np.int64), np.zeros((0, 4), F32), 10, 2, owner, 2)
    assert r["n_uniq"] == 0 and list(r["dest_counts"]) == [0, 0]
    r = orc.sort_dedup_route(np.array([9]), np.ones((1, 4), F32), 10, 2, owner, 2)
    assert r["n_uniq"] == 1 and r["dest_counts"].sum() == 1


@pytest.mark.parametrize("opt", ["sgd", "adagrad", "adam"])
def test_sparse_step_vs_float64(opt):
    rng = np.random.default_rng(2)
    V, D, n, P, T = 400, 8, 3, 5, 600
    hpar = {"lr": 0.1, "beta1": 0.9, "beta2": 0.999, "eps": 1e-8}
    st = orc.init_state(opt, V, D, seed=3)
    ref = {k: v.astype(np.float64) for k, v in st.items()}
    batches = [(rng.integers(0, V, T), rng.standard_normal((T, D), dtype=F32)) for _ in range(n)]
    owner = orc.owner_table("embedding", P, n)
    res = orc.sparse_step(st, opt, hpar, 1, batches, V, P, owner, "mean")
    g = np.zeros((V, D))
    for ids, vals in batches:
        np.add.at(g, ids, vals.astype(np.float64))
    g /= n
    touched = np.unique(np.concatenate([b[0] for b in batches]))
    gt = g[touched]
    if opt == "sgd":
        ref["w"][touched] -= 0.1 * gt
    elif opt == "adagrad":
        ref["acc"][touched] += gt * gt
        ref["w"][touched] -= 0.1 * gt / np.sqrt(ref["acc"][touched])
    else:
        m = 0.1 * gt
        v = 0.001 * gt * gt
        lr_t = 0.1 * np.sqrt(1 - 0.999) / (1 - 0.9)
        ref["w"][touched] -= lr_t * m / (np.sqrt(v) + 1e-8)
    assert np.allclose(st["w"], ref["w"], rtol=1e-5, atol=1e-6)
    untouched = np.setdiff1d(np.arange(V), touched)
    assert np.array_equal(st["w"][untouched], orc.init_rows(0, V, D, 3)[untouched])
    for r, (ids, _) in enumerate(batches):
        assert np.array_equal(res[r]["out"], st["w"][ids])


def test_init_rows_range_and_determinism():
    a = orc.init_rows(10, 20, 16, seed=5)
    b = orc.init_rows(0, 30, 16, seed=5)[10:20]
    assert np.array_equal(a, b)
    assert a.min() >= -0.05 and a.max() < 0.05 and a.dtype == F32
    assert not np.array_equal(a, orc.init_rows(10, 20, 16, seed=6))


def test_owner_table_matches_planner():
    for n in (1, 2, 4, 8):
        g = hp.GraphSpec("g", (hp.VariableSpec("softmax", 800_000, 2048, 0.01, "sparse", True),), 0)
        plan = hp.transform_ps(g, hp.ClusterSpec.b200_box(n), partitions={"softmax": 16})
        assert np.array_equal(plan.owner_table("softmax"), orc.owner_table("softmax", 16, n))


@pytest.mark.parametrize("T,D,V,n,P", [(1, 4, 10, 1, 1), (0, 4, 10, 2, 2), (500, 8, 50, 2, 4),
                                       (3000, 16, 40, 3, 5), (20000, 64, 100000, 4, 8),
                                       (40000, 8, 7, 1, 1)])
def test_c_oracle_bit_exact_vs_numpy(T, D, V, n, P):
    """oracle/hp_oracle.c (the multithreaded CPU baseline) == oracle.py, bit for bit."""
    from oracle import coracle as co

    rng = np.random.default_rng(T + D)
    own = orc.owner_table("emb", P, n)
    ids = rng.integers(0, V, T)
    vals = rng.standard_normal((T, D)).astype(F32)
    a = orc.sort_dedup_route(ids, vals, V, P, own, n)
    b = co.sort_dedup_route(ids, vals, V, P, own, n)
    for k in ("send_ids", "send_rows", "counts", "inv", "dest_counts", "n_uniq"):
        assert np.array_equal(a[k], b[k]), k
    for opt in ("sgd", "adagrad", "adam"):
        s1 = orc.init_state(opt, V, D, 3)
        s2 = {k: v.copy() for k, v in s1.items()}
        bs = [(rng.integers(0, V, T), rng.standard_normal((T, D)).astype(F32)) for _ in range(n)]
        r1 = orc.sparse_step(s1, opt, {"lr": 0.1}, 3, bs, V, P, own)
        r2 = co.sparse_step(s2, opt, {"lr": 0.1}, 3, bs, V, P, own)
        for k in s1:
            assert np.array_equal(s1[k], s2[k]), (opt, k)
        for x, y in zip(r1, r2):
            assert np.array_equal(x["out"], y["out"])


def test_ar_sparse_step_is_one_worker_step_over_the_concatenation():
    """AR for a sparse Weight = the concatenated slices applied once, scaled by 1/n."""
    rng = np.random.default_rng(3)
    V, D, n, T = 500, 8, 3, 200
    batches = [(rng.integers(0, V, T), rng.standard_normal((T, D)).astype(F32)) for _ in range(n)]
    a = orc.init_state("adagrad", V, D, 1)
    b = {k: v.copy() for k, v in a.items()}
    res = orc.ar_sparse_step(a, "adagrad", {"lr": 0.1}, 1, batches)
    ids = np.concatenate([x[0] for x in batches])
    vals = np.concatenate([x[1] for x in batches])
    uniq, sums, _, _ = orc.grouped_tree_sum(ids, vals)
    orc.apply_rows("adagrad", b, uniq, sums * F32(1.0 / n), {"lr": 0.1}, 1)
    for k in a:
        assert np.array_equal(a[k], b[k])
    for r, (i, _) in enumerate(batches):
        assert np.array_equal(res[r]["out"], b["w"][i])


def test_out_of_range_ids_are_dropped_numpy_and_c():
    """Ids outside [0, V) update nothing, pull a zero row and get inv = -1, in
    both oracles (the device drops them the same way, never clamps)."""
    from oracle import coracle

    rng = np.random.default_rng(9)
    V, D, P, n, T = 1000, 8, 4, 2, 600
    ids = rng.integers(0, V, T)
    bad = rng.choice(T, 40, replace=False)
    ids[bad[:20]] = V + rng.integers(0, 5, 20)
    ids[bad[20:]] = -1 - rng.integers(0, 5, 20)
    vals = rng.standard_normal((T, D), dtype=F32)
    owner = orc.owner_table("embedding", P, n)
    ok = (ids >= 0) & (ids < V)
    a = orc.sort_dedup_route(ids, vals, V, P, owner, n)
    b = coracle.sort_dedup_route(ids, vals, V, P, owner, n)
    ref = orc.sort_dedup_route(ids[ok], vals[ok], V, P, owner, n)
    for r in (a, b):
        assert r["n_uniq"] == ref["n_uniq"]
        assert np.array_equal(r["send_ids"], ref["send_ids"])
        assert np.array_equal(r["send_rows"], ref["send_rows"])
        assert np.array_equal(r["inv"][ok], ref["inv"])
        assert np.all(r["inv"][~ok] == -1)
        assert np.array_equal(r["dest_counts"], ref["dest_counts"])
    states = [orc.init_state("adagrad", V, D, 3) for _ in range(3)]
    hpar = {"lr": 0.1}
    r1 = orc.sparse_step(states[0], "adagrad", hpar, 1, [(ids, vals)], V, P, np.zeros(P, np.int32))
    r2 = coracle.sparse_step(states[1], "adagrad", hpar, 1, [(ids, vals)], V, P, np.zeros(P, np.int32))
    r3 = orc.sparse_step(states[2], "adagrad", hpar, 1, [(ids[ok], vals[ok])], V, P, np.zeros(P, np.int32))
    assert np.array_equal(states[0]["w"], states[2]["w"])
    assert np.array_equal(states[1]["w"], states[2]["w"])
    for r in (r1, r2):
        assert np.array_equal(r[0]["out"][ok], r3[0]["out"])
        assert not r[0]["out"][~ok].any()
