"""Planner parity: routing, classification, placement and the P search.

Every case is pinned two ways: against golden vectors produced by the
reference itself (tests/golden/make_golden.py, committed) and, when
/root/reference exists, against the live reference on the same inputs.
"""

import json
import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1808_02621_b200 as hp
from golden.make_golden import cases, evaluator, plan_digest
from oracle import oracle as orc


def _graph(golden, name):
    return hp.load_graph_spec(golden["fixtures"][name])


# ------------------------------------------------------------------ routing
def test_even_split_golden(golden):
    for total, parts, sizes in golden["even_split"]:
        assert hp.even_split(total, parts) == sizes
        assert orc.even_split(total, parts) == sizes


def test_partition_sizes_golden(golden):
    for total, parts, exp in golden["partition_sizes"]:
        v = hp.VariableSpec("e", total, 4, 0.01, "sparse", True)
        sizes = [e for _, e in hp.partition_variable(v, parts).partitions]
        got = sizes if parts <= 64 else [min(sizes), max(sizes), sum(sizes)]
        assert got == exp


def test_partition_known_answers():
    # reference tests/test_model.py:151-180
    sv = lambda n: hp.VariableSpec("e", n, 4, 0.1, "sparse", True)
    assert hp.partition_variable(sv(10), 1).partitions == ((0, 10),)
    assert [e for _, e in hp.partition_variable(sv(10), 4).partitions] == [3, 3, 2, 2]
    assert {e for _, e in hp.partition_variable(sv(800_000), 128).partitions} == {6250}
    with pytest.raises(hp.SpecError, match="not partitionable"):
        hp.partition_variable(hp.VariableSpec("w", 1000, 4, 1.0, "dense"), 2)
    with pytest.raises(hp.SpecError, match="partition count"):
        hp.partition_variable(sv(10), 11)


@settings(max_examples=200, deadline=None)
@given(st.integers(1, 10**7), st.integers(1, 4096), st.integers(0, 2**31 - 1))
def test_closed_form_router_matches_bounds(V, P, seed):
    """The closed form the CUDA router evaluates == search in the even-split bounds."""
    P = min(P, V)
    rng = np.random.default_rng(seed)
    rows = np.concatenate([rng.integers(0, V, 256), [0, V - 1],
                           hp.partition_bounds(V, P)[1:-1], hp.partition_bounds(V, P)[1:-1] - 1])
    rows = np.clip(rows, 0, V - 1)
    assert np.array_equal(hp.partition_of_row(rows, V, P), orc.partition_of(rows, V, P))


def test_hash_start_golden(golden):
    from paper_1808_02621_b200.placement import _hash_start

    for name, m, start in golden["hash_start"]:
        assert _hash_start(name, m) == start
        assert orc.owner_table(name, 1, m)[0] == start


# ------------------------------------------------------------------ classification
def test_assign_mechanism_golden(golden):
    for kind, alpha, ea, ep, m, mech in golden["assign_mechanism"]:
        v = hp.VariableSpec("v", 1000, 4, alpha, kind, kind == "sparse")
        got = hp.assign_mechanism(v, hp.ClusterSpec(m, 1, 100.0), hp.MechanismPolicy(ea, ep))
        assert got.value == mech


def test_single_box_mapping(golden):
    """one box of n GPUs == ClusterSpec(n, 1); embedding -> PS with
    owners (crc32('embedding') % 8 + p) % 8."""
    g = _graph(golden, "lm")
    plan = hp.transform_hybrid(g, hp.ClusterSpec.b200_box(8), partitions={"embedding": 16})
    assert plan.mech_of["lstm"] is hp.Mechanism.AR
    assert plan.mech_of["embedding"] is hp.Mechanism.PS
    assert list(plan.owner_table("embedding")) == [(6 + p) % 8 for p in range(16)]
    one = hp.transform_hybrid(g, hp.ClusterSpec.b200_box(1), partitions={"embedding": 16})
    assert one.mech_of["embedding"] is hp.Mechanism.AR and one.partitions_of["embedding"] == 1


# ------------------------------------------------------------------ placement
def test_plans_golden(golden):
    n = 0
    for case in golden["plans"]:
        g = _graph(golden, case["graph"])
        c = hp.ClusterSpec(case["machines"], case["gpus"], 100.0)
        sparse = [v.name for v in g.variables if v.kind == "sparse" and v.partitionable]
        pm = {k: case["P"] for k in sparse} or None
        if case["arch"] == "hybrid":
            plan = hp.transform_hybrid(g, c, partitions=pm)
        elif case["arch"] == "ps_opt":
            plan = hp.transform_ps(g, c, partitions=pm)
        else:
            plan = hp.transform_ar(g, c)
        assert plan_digest(hp.plan_to_dict(plan)) == case["dict"], case["graph"]
        for var, owners in case["owners"].items():
            assert list(plan.owner_table(var)) == owners
            if case["gpus"] == 1 and plan.partitions_of[var] > 1:
                assert list(orc.owner_table(var, len(owners), case["machines"])) == owners
        assert hp.validate_plan(plan, g, c) == case["valid"]
        n += 1
    assert n > 100


def test_mixed_placement_golden(golden):
    g = hp.GraphSpec("mix", (
        hp.VariableSpec("a", 1000, 4, 0.1, "sparse", True),
        hp.VariableSpec("b", 5000, 4, 0.1, "sparse", False),
        hp.VariableSpec("c", 3000, 8, 0.2, "sparse", True),
        hp.VariableSpec("d", 700, 4, 1.0, "dense"),
        hp.VariableSpec("f", 9000, 4, 0.3, "sparse", False),
    ), 0.0)
    for case in golden["mixed_plans"]:
        c = hp.ClusterSpec(case["machines"], 1, 50.0)
        plan = hp.transform_ps(g, c, partitions={"a": case["pa"], "c": 4})
        assert hp.plan_to_dict(plan) == case["dict"]
        assert hp.plan_to_dict(hp.plan_from_dict(case["dict"])) == case["dict"]


def test_dense_only_isomorphic_to_ar(golden):
    g = _graph(golden, "resnet50")
    c = hp.load_cluster_spec(golden["fixtures"]["cluster8x6"])
    assert hp.transform_hybrid(g, c).node_multiset() == hp.transform_ar(g, c).node_multiset()


def test_validate_fault_injection(golden):
    from dataclasses import replace

    g = _graph(golden, "lm")
    c = hp.ClusterSpec(4, 1, 100.0)
    plan = hp.transform_hybrid(g, c, partitions={"embedding": 8})
    assert hp.validate_plan(plan, g, c) == []
    nodes = list(plan.nodes)
    i = next(k for k, nd in enumerate(nodes) if nd.role == "update")
    nodes[i] = replace(nodes[i], machine=(nodes[i].machine + 1) % 4)
    bad = replace(plan, nodes=tuple(nodes))
    assert any("not colocated" in p for p in hp.validate_plan(bad, g, c))
    assert any("chief" in p for p in hp.validate_plan(replace(plan, chief=(9, 0)), g, c))


# ------------------------------------------------------------------ P search
def test_fit_and_optimal_golden(golden):
    for name, case in golden["fits"].items():
        prm = hp.fit_theta([tuple(s) for s in case["samples"]])
        for a, b in zip([prm.theta0, prm.theta1, prm.theta2], case["theta"]):
            assert a == pytest.approx(b, rel=1e-9, abs=1e-9), name
        assert hp.optimal_p(prm) == case["best_p"], name


def test_search_golden(golden):
    for name, case in golden["searches"].items():
        ev = evaluator(case["kind"])
        got = hp.sample_search(ev, case["start"], case["threshold"], case["max_p"])
        assert [list(s) for s in got] == case["samples"], name
        res = hp.tune_evaluator(ev, case["start"], case["threshold"], case["max_p"]).to_dict()
        assert res["best_p"] == case["result"]["best_p"], name
        assert res["samples_taken"] == case["result"]["samples_taken"]
        assert res["predicted_time_us"] == pytest.approx(case["result"]["predicted_time_us"],
                                                         rel=1e-9)


def test_tuner_known_answers():
    # reference tests/test_tuning.py:124-199 and test_acceptance.py:169-194
    samples = hp.sample_search(lambda p: 10 + 1000 / p + 0.1 * p, start_p=8)
    assert [p for p, _ in samples] == [4, 8, 16, 32, 64, 128]
    assert [p for p, _ in hp.sample_search(lambda p: 42.0, start_p=8)] == [4, 8, 16]
    assert [p for p, _ in hp.sample_search(lambda p: float(p), start_p=8)] == [1, 2, 4, 8, 16]
    res = hp.tune_evaluator(lambda p: 10 + 1000 / p + 0.1 * p, start_p=8)
    assert res.best_p == 100 and res.samples_taken <= 12
    assert res.predicted_time == pytest.approx(30.0, rel=1e-6)
    with pytest.raises(hp.TuningError, match="P=8"):
        hp.sample_search(lambda p: 1 / 0, start_p=8)
    with pytest.raises(hp.TuningError, match="3 distinct"):
        hp.fit_theta([(4, 1.0), (4, 1.1), (8, 2.0)])
    paper = [50.5e3, 78.6e3, 96.5e3, 96.1e3, 98.9e3, 93.2e3]
    prm = hp.fit_theta([(8 * 2 ** i, 1e6 / t) for i, t in enumerate(paper)])
    assert hp.optimal_p(prm) == 87  # BASELINE.md tuner golden


def test_tune_uses_measure_callback(golden):
    g = _graph(golden, "lm")
    c = hp.ClusterSpec.b200_box(8)
    seen = []

    def measure(plan, iterations):
        p = plan.partitions_of["embedding"]
        seen.append((p, iterations))
        return 10 + 1000 / p + 0.1 * p

    res = hp.tune(g, c, lambda p: hp.transform_hybrid(g, c, partitions={"embedding": p}),
                  measure, iterations=10)
    assert res.best_p == 100 and seen[0] == (8, 10)


# ------------------------------------------------------------------ live reference
def test_live_reference_parity(reference):
    sp = reference
    _, split, clusters, names, parts, mech, fits, searches = cases()
    for t, p in split:
        assert hp.even_split(t, p) == sp.model.even_split(t, p)
    rng = np.random.default_rng(7)
    for _ in range(200):
        m = int(rng.integers(1, 9))
        nvar = int(rng.integers(1, 5))
        vs = []
        for k in range(nvar):
            kind = "dense" if rng.random() < 0.3 else "sparse"
            alpha = 1.0 if kind == "dense" else float(rng.uniform(0.001, 1.0))
            vs.append((f"v{k}", int(rng.integers(1, 5000)), int(rng.integers(1, 64)), alpha, kind,
                       bool(rng.random() < 0.7)))
        mine = hp.GraphSpec("g", tuple(hp.VariableSpec(*v) for v in vs), 0.0)
        ref = sp.GraphSpec("g", tuple(sp.VariableSpec(*v) for v in vs), 0.0)
        parts_ = {v[0]: int(rng.integers(1, min(v[1], 40) + 1)) for v in vs
                  if v[5] and v[4] == "sparse"}
        pol = (float(rng.uniform(0.5, 2)), float(rng.uniform(0.5, 2)))
        a = hp.transform_hybrid(mine, hp.ClusterSpec(m, 1, 10.0), hp.MechanismPolicy(*pol), parts_)
        b = sp.transform_hybrid(ref, sp.ClusterSpec(m, 1, 10.0), sp.MechanismPolicy(*pol), parts_)
        assert hp.plan_to_dict(a) == sp.plan_to_dict(b)


def test_transfer_model_golden(golden):
    """Predicted per-GPU bytes (reference transfer_model) of the
    one-box hybrid plans, against the reference's own outputs."""
    assert golden["transfer"]
    for case in golden["transfer"]:
        g = _graph(golden, case["graph"])
        c = hp.ClusterSpec(case["machines"], 1, 7200.0)
        sparse = [v.name for v in g.variables if v.kind == "sparse"]
        plan = hp.transform_hybrid(g, c, partitions={n: 8 for n in sparse})
        assert hp.transfer_model(g, plan, c).to_rows() == case["rows"]


def test_transfer_model_live(reference):
    sp = reference
    rng = np.random.default_rng(3)
    for _ in range(100):
        m, G = int(rng.integers(1, 7)), int(rng.integers(1, 3))
        vs = []
        for k in range(int(rng.integers(1, 5))):
            kind = "dense" if rng.random() < 0.3 else "sparse"
            alpha = 1.0 if kind == "dense" else float(rng.uniform(0.001, 1.0))
            vs.append((f"v{k}", int(rng.integers(1, 5000)), int(rng.integers(1, 64)), alpha, kind,
                       bool(rng.random() < 0.7)))
        parts = {v[0]: int(rng.integers(1, min(v[1], 40) + 1)) for v in vs
                 if v[5] and v[4] == "sparse"}
        mine = hp.GraphSpec("g", tuple(hp.VariableSpec(*v) for v in vs), 0.0)
        ref = sp.GraphSpec("g", tuple(sp.VariableSpec(*v) for v in vs), 0.0)
        for arch in ("ar", "ps_naive", "ps_opt", "hybrid"):
            cm, cr = hp.ClusterSpec(m, G, 10.0), sp.ClusterSpec(m, G, 10.0)
            if arch == "ar":
                a, b = hp.transform_ar(mine, cm), sp.transform_ar(ref, cr)
            elif arch == "hybrid":
                a, b = hp.transform_hybrid(mine, cm, None, parts), sp.transform_hybrid(ref, cr, None, parts)
            else:
                la = arch == "ps_opt"
                a = hp.transform_ps(mine, cm, local_agg=la, partitions=parts)
                b = sp.transform_ps(ref, cr, local_agg=la, partitions=parts)
            got = hp.transfer_model(mine, a, cm).to_rows()
            want = sp.transfer_model(ref, b, cr).to_rows()
            assert np.allclose([[r["egress_bytes"], r["ingress_bytes"]] for r in got],
                               [[r["egress_bytes"], r["ingress_bytes"]] for r in want], rtol=1e-12)


def test_tune_reference_signature(golden):
    """tune(graph, cluster, plan_builder, profile, threshold, iterations, seed):
    the reference's positional form; the profile's compute time is added to
    every measured sample (a constant: the argmin is unchanged)."""
    g = _graph(golden, "lm")
    c = hp.ClusterSpec.b200_box(8)

    def measure(plan, iterations):
        return 10 + 1000 / plan.partitions_of["embedding"] + 0.1 * plan.partitions_of["embedding"]

    build = lambda p: hp.transform_hybrid(g, c, partitions={"embedding": p})  # noqa: E731
    res = hp.tune(g, c, build, hp.ComputeProfile(compute_us_per_gpu=50.0), 0.10, 10, 0,
                  measure=measure)
    base = hp.tune(g, c, build, hp.ComputeProfile(), measure=measure)
    assert res.best_p == base.best_p == 100
    assert res.predicted_time == pytest.approx(base.predicted_time + 50.0)
    with pytest.raises(hp.SpecError):
        hp.ComputeProfile(compute_us_per_gpu=-1)
