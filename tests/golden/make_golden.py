"""Generate planner golden vectors by importing the REFERENCE package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``sparseplan`` from /root/reference/pkg/src (read-only; nothing is
copied) and records the outputs of its routing / classification / placement /
search functions on a fixed case list into ``planner_golden.json``. The GPU box
has no /root/reference, so the tests compare against this committed file; when
the reference is present they also re-run it live.
"""

from __future__ import annotations

import hashlib
import json
import math
import sys
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
REF_FIX = Path("/root/reference/pkg/fixtures")
OUT = Path(__file__).resolve().parent / "planner_golden.json"


def _import_ref():
    sys.dont_write_bytecode = True
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import sparseplan  # noqa: F401

    return sparseplan


def cases():
    """Inputs shared by the generator and the parity test."""
    fixtures = {n: (REF_FIX / f"{n}.json").read_text() if REF_FIX.exists() else None
                for n in ("lm", "nmt", "resnet50", "cluster8x6")}
    split = [(10, 1), (10, 4), (800_000, 128), (813_300_000, 8), (37_000, 16), (7, 7), (1, 1),
             (10_000_000, 128), (10_000, 2), (74_900_000, 24), (1_280_000, 48), (5, 3)]
    clusters = [(1, 1), (2, 1), (4, 1), (8, 1), (8, 6), (3, 1), (1, 4)]
    names = ["embedding", "softmax", "emb_enc", "emb_dec", "embeddings", "e", "w"]
    parts = [1, 2, 4, 8, 11, 12, 16, 32, 64, 128]
    mech = [(kind, alpha, eff_ar, eff_ps, m)
            for kind in ("dense", "sparse")
            for alpha in ((1.0,) if kind == "dense" else (0.001, 0.02, 0.5, 0.83, 0.99, 1.0))
            for eff_ar, eff_ps in ((1.0, 1.0), (1.0, 1.2), (0.9, 1.0), (2.0, 0.5))
            for m in (1, 2, 8)]
    paper_lm = [50.5e3, 78.6e3, 96.5e3, 96.1e3, 98.9e3, 93.2e3]
    paper_nmt = [90.7e3, 97.0e3, 96.5e3, 101.6e3, 98.5e3, 100.0e3]
    fits = {
        "synthetic": [(p, 10 + 1000 / p + 0.1 * p) for p in (1, 2, 4, 8, 16, 64)],
        "flat": [(1, 50.0), (2, 50.0), (4, 50.0), (8, 50.0)],
        "decreasing": [(p, 100.0 / p) for p in (1, 2, 4, 8)],
        "increasing": [(p, 5.0 * p) for p in (1, 2, 4, 8)],
        "paper_lm": [(8 * 2 ** i, 1e6 / t) for i, t in enumerate(paper_lm)],
        "paper_nmt": [(8 * 2 ** i, 1e6 / t) for i, t in enumerate(paper_nmt)],
        "noisy": [(4, 31.2), (8, 20.5), (16, 17.9), (32, 19.4), (64, 26.0)],
    }
    searches = {
        "convex_8": ("convex", 8, 0.10, 1 << 20),
        "convex_1": ("convex", 1, 0.10, 1 << 20),
        "convex_300": ("convex", 300, 0.10, 1 << 20),
        "const_8": ("const", 8, 0.10, 1 << 20),
        "increasing_8": ("linear", 8, 0.10, 1 << 20),
        "cap_32": ("inverse", 8, 0.10, 32),
        "thr0": ("slow", 1, 0.0, 8),
        "convex_thr25": ("convex", 4, 0.25, 1 << 20),
        "paper_lm_table": ("paper_lm", 8, 0.10, 256),
    }
    return fixtures, split, clusters, names, parts, mech, fits, searches


def plan_digest(d: dict) -> dict:
    """Compact form of plan_to_dict: small fields verbatim, node list hashed."""
    nodes = json.dumps(d["nodes"], sort_keys=True, separators=(",", ":"))
    return {k: v for k, v in d.items() if k != "nodes"} | {
        "n_nodes": len(d["nodes"]), "nodes_sha256": hashlib.sha256(nodes.encode()).hexdigest()}


def evaluator(kind: str):
    lm = dict(zip([8, 16, 32, 64, 128, 256], [50.5e3, 78.6e3, 96.5e3, 96.1e3, 98.9e3, 93.2e3]))
    table = {
        "convex": lambda p: 10 + 1000 / p + 0.1 * p,
        "const": lambda p: 42.0,
        "linear": lambda p: float(p),
        "inverse": lambda p: 1000.0 / p,
        "slow": lambda p: 100.0 - 0.001 * p,
        "paper_lm": lambda p: 1e6 / lm.get(p, lm[min(lm, key=lambda q: abs(math.log2(q / p)))]),
    }
    return table[kind]


def generate(sp) -> dict:
    fixtures, split, clusters, names, parts, mech, fits, searches = cases()
    out: dict = {"fixtures": fixtures}
    out["even_split"] = [[t, p, sp.model.even_split(t, p)] for t, p in split if p <= 64]
    out["partition_sizes"] = []
    for t, p in split:
        v = sp.VariableSpec("e", t, 4, 0.01, "sparse", True)
        ps = sp.partition_variable(v, p)
        sizes = [e for _, e in ps.partitions]
        out["partition_sizes"].append([t, p, sizes if p <= 64 else [min(sizes), max(sizes),
                                                                    sum(sizes)]])
    out["hash_start"] = [[n, m, sp.placement._hash_start(n, m)] for n in names
                         for m in (1, 2, 3, 4, 6, 8)]
    out["assign_mechanism"] = []
    for kind, alpha, ea, ep, m in mech:
        v = sp.VariableSpec("v", 1000, 4, alpha, kind, kind == "sparse")
        c = sp.ClusterSpec(m, 1, 100.0)
        out["assign_mechanism"].append(
            [kind, alpha, ea, ep, m, sp.assign_mechanism(v, c, sp.MechanismPolicy(ea, ep)).value])
    # plans for the fixture graphs on each cluster shape and P
    out["plans"] = []
    for gname in ("lm", "nmt", "resnet50"):
        if fixtures[gname] is None:
            continue
        g = sp.load_graph_spec(fixtures[gname])
        sparse = [v.name for v in g.variables if v.kind == "sparse" and v.partitionable]
        for m, gp in clusters:
            c = sp.ClusterSpec(m, gp, 100.0)
            for p in parts:
                pm = {n: p for n in sparse} or None
                for arch in ("hybrid", "ps_opt", "ar"):
                    if arch == "hybrid":
                        plan = sp.transform_hybrid(g, c, partitions=pm)
                    elif arch == "ps_opt":
                        plan = sp.transform_ps(g, c, partitions=pm)
                    else:
                        if p != 1:
                            continue
                        plan = sp.transform_ar(g, c)
                    owners = {n: [plan.owner_of(n, i) for i in range(plan.partitions_of[n])]
                              for n in plan.partitions_of
                              if plan.mech_of[n] == sp.Mechanism.PS}
                    out["plans"].append({
                        "graph": gname, "machines": m, "gpus": gp, "P": p, "arch": arch,
                        "dict": plan_digest(sp.plan_to_dict(plan)), "owners": owners,
                        "valid": sp.validate_plan(plan, g, c),
                    })
    # multi-variable placement (greedy unpartitioned + round-robin partitioned)
    g = sp.GraphSpec("mix", (
        sp.VariableSpec("a", 1000, 4, 0.1, "sparse", True),
        sp.VariableSpec("b", 5000, 4, 0.1, "sparse", False),
        sp.VariableSpec("c", 3000, 8, 0.2, "sparse", True),
        sp.VariableSpec("d", 700, 4, 1.0, "dense"),
        sp.VariableSpec("f", 9000, 4, 0.3, "sparse", False),
    ), 0.0)
    out["mixed_plans"] = []
    for m in (2, 3, 5, 8):
        c = sp.ClusterSpec(m, 1, 50.0)
        for pa in (1, 3, 7):
            plan = sp.transform_ps(g, c, partitions={"a": pa, "c": 4})
            out["mixed_plans"].append({"machines": m, "pa": pa, "dict": sp.plan_to_dict(plan)})
    # tuner
    out["fits"] = {}
    for name, samples in fits.items():
        prm = sp.fit_theta(samples)
        out["fits"][name] = {"samples": samples, "theta": [prm.theta0, prm.theta1, prm.theta2],
                             "best_p": sp.optimal_p(prm)}
    out["searches"] = {}
    for name, (kind, start, thr, max_p) in searches.items():
        res = sp.tune_evaluator(evaluator(kind), start, thr, max_p)
        out["searches"][name] = {
            "kind": kind, "start": start, "threshold": thr, "max_p": max_p,
            "samples": sp.sample_search(evaluator(kind), start, thr, max_p),
            "result": res.to_dict(),
        }
    # transfer model of the one-box mapping (predicted exchange bytes)
    out["transfer"] = []
    if fixtures["lm"] is not None:
        for gname in ("lm", "nmt"):
            gg = sp.load_graph_spec(fixtures[gname])
            for m in (2, 4, 8):
                c = sp.ClusterSpec(m, 1, 7200.0)
                sparse = [v.name for v in gg.variables if v.kind == "sparse"]
                plan = sp.transform_hybrid(gg, c, partitions={n: 8 for n in sparse})
                out["transfer"].append({"graph": gname, "machines": m,
                                        "rows": sp.transfer_model(gg, plan, c).to_rows()})
    return out


if __name__ == "__main__":
    sp = _import_ref()
    doc = generate(sp)
    OUT.write_text(json.dumps(doc, sort_keys=True, separators=(",", ":")))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")
