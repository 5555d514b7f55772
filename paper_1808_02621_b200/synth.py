"""Synthetic inputs of the BASELINE.json shapes.

Seeds: ``default_rng(seed * 1000 + rank)`` per rank. Row ids are bounded
Zipf(s) over [0, V) with P(k) proportional to (k+1)^-s and frequency-ranked ids
(0 = hottest, as in a sorted vocabulary); sampled-softmax negatives are
log-uniform, P(k) = log((k+2)/(k+1)) / log(V+1). Gradient values are standard
normal fp32.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np


@lru_cache(maxsize=8)
def _zipf_cdf(V: int, s: float) -> np.ndarray:
    w = np.arange(1, V + 1, dtype=np.float64) ** (-s)
    c = np.cumsum(w)
    return c / c[-1]


def zipf_ids(rng: np.random.Generator, V: int, n: int, s: float = 1.1) -> np.ndarray:
    u = rng.random(n)
    return np.minimum(np.searchsorted(_zipf_cdf(V, s), u, side="right"), V - 1).astype(np.int64)


def log_uniform_ids(rng: np.random.Generator, V: int, n: int) -> np.ndarray:
    k = np.floor(np.exp(rng.random(n) * np.log(V + 1.0))).astype(np.int64) - 1
    return np.clip(k, 0, V - 1)


@dataclass
class TableShape:
    name: str
    V: int
    D: int
    T: int                 # ids per worker per step
    sampled: int = 0       # extra shared log-uniform ids (sampled softmax)
    zipf_s: float = 1.1


@dataclass
class Workload:
    name: str
    tables: list
    dense: dict            # name -> elements
    optimizer: dict
    words_per_worker: int  # words/s numerator per worker per step
    partitions: int = 8
    notes: str = ""
    extra: dict = field(default_factory=dict)

    def graph_json(self) -> dict:
        """A reference-schema graph document (`sparseplan/model.py:241-271`)."""
        vars_ = [{"name": n, "elements": e, "elem_bytes": 4, "alpha": 1, "kind": "dense"}
                 for n, e in self.dense.items()]
        for t in self.tables:
            alpha = min(1.0, (t.T + t.sampled) / t.V)
            vars_.append({"name": t.name, "elements": t.V, "elem_bytes": 4 * t.D,
                          "alpha": alpha, "kind": "sparse", "partitionable": True})
        return {"name": self.name, "batch_per_gpu": 128, "compute_us_per_gpu": 0.0,
                "variables": vars_}


WORKLOADS = {
    "tiny": Workload("tiny", [TableShape("embedding", 10_000, 128, 2560)],
                     {"dense": 256 * 256 + 256}, {"kind": "sgd", "lr": 0.1}, 2560, partitions=2),
    "lm1b": Workload("lm1b", [TableShape("embedding", 800_000, 512, 2560),
                              TableShape("softmax", 800_000, 512, 2560, sampled=8192)],
                     {"lstm": 9_400_000}, {"kind": "adagrad", "lr": 0.2, "init_acc": 0.1}, 2560,
                     partitions=8),
    "nmt": Workload("nmt", [TableShape("emb_enc", 37_000, 1024, 2560),
                            TableShape("emb_dec", 37_000, 1024, 2560)],
                    {"lstm_stack": 94_100_000},
                    {"kind": "adam", "lr": 1e-3, "beta1": 0.9, "beta2": 0.999, "eps": 1e-8},
                    2560, partitions=8),
    "dense": Workload("dense", [], {"conv_fc": 25_600_000}, {"kind": "sgd", "lr": 0.1}, 0),
}
# diagnosis variants of the LM1B step: only its sparse tables / only its dense part
WORKLOADS["lm1b_sparse"] = Workload("lm1b_sparse", WORKLOADS["lm1b"].tables, {},
                                    WORKLOADS["lm1b"].optimizer, 2560, partitions=8)
WORKLOADS["lm1b_dense"] = Workload("lm1b_dense", [], dict(WORKLOADS["lm1b"].dense),
                                   WORKLOADS["lm1b"].optimizer, 2560, partitions=8)


def micro_workload(draws: int) -> Workload:
    """10M x 128 table, Zipf(1.1); alpha is calibrated by the draw count."""
    return Workload(f"micro_{draws}", [TableShape("embedding", 10_000_000, 128, draws)], {},
                    {"kind": "adagrad", "lr": 0.2, "init_acc": 0.1}, 0, partitions=8)


def make_sparse_batch(t: TableShape, rng: np.random.Generator):
    ids = zipf_ids(rng, t.V, t.T, t.zipf_s)
    if t.sampled:
        ids = np.concatenate([ids, log_uniform_ids(rng, t.V, t.sampled)])
    vals = rng.standard_normal((ids.size, t.D), dtype=np.float32)
    return ids, vals


def make_batch(w: Workload, seed: int, rank: int, dense: bool = True) -> dict:
    rng = np.random.default_rng(seed * 1000 + rank)
    out = {t.name: make_sparse_batch(t, rng) for t in w.tables}
    if dense:
        for name, n in w.dense.items():
            out[name] = rng.standard_normal(n, dtype=np.float32)
    return out


def graph_batches(graph, seed: int, rank: int, count: int, device) -> list:
    """Device batches shaped by a planner GraphSpec (the reference's inputs):
    a sparse Weight gets ceil-rounded alpha * V Zipf(1.1) ids of its row width,
    a dense Weight a standard-normal gradient of its element count."""
    import torch

    out = []
    for i in range(count):
        rng = np.random.default_rng((seed + i) * 1000 + rank)
        b = {}
        for v in graph.variables:
            if v.kind == "sparse":
                D = v.elem_bytes // 4
                T = max(1, int(round(v.alpha * v.elements)))
                ids = zipf_ids(rng, v.elements, T)
                vals = rng.standard_normal((T, D), dtype=np.float32)
                b[v.name] = (torch.from_numpy(ids).to(device), torch.from_numpy(vals).to(device))
            else:
                b[v.name] = torch.from_numpy(rng.standard_normal(v.elements, dtype=np.float32)).to(device)
        out.append(b)
    return out
