"""ctypes front of oracle/hp_oracle.c (TEST INFRASTRUCTURE ONLY).

Same functions and results as :mod:`oracle.oracle` (bit-exact, checked in
tests/test_oracle.py), multithreaded with OpenMP so bench.py's CPU baseline
and ``--impl reference`` use every host core. Built by ``make -C oracle``
(``__graft_entry__.build()`` runs it).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from . import oracle as orc

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "build", "libhp_oracle.so")
_lib = None

F32 = np.float32


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = C.CDLL(_SO)
        vp, i64, i32, f = C.c_void_p, C.c_int64, C.c_int32, C.c_float
        L.hpo_sort_dedup_route.restype = i64
        L.hpo_sort_dedup_route.argtypes = [vp, vp, i64, C.c_int, i64, i32, vp, i32,
                                           vp, vp, vp, vp, vp]
        L.hpo_merge_apply.restype = i64
        L.hpo_merge_apply.argtypes = [vp, vp, i64, C.c_int, C.c_int, vp, vp, vp,
                                      f, f, f, f, f, f, f, f]
        L.hpo_gather.restype = None
        L.hpo_gather.argtypes = [vp, i64, vp, i64, C.c_int, vp]
        L.hpo_dense_mean.restype = None
        L.hpo_dense_mean.argtypes = [vp, C.c_int, i64, f, vp]
        L.hpo_chunk.restype = C.c_int
        L.hpo_set_threads.restype = C.c_int
        L.hpo_set_threads.argtypes = [C.c_int]
        L.hpo_set_threads(os.cpu_count() or 1)  # every host thread (torchrun sets OMP=1)
        assert L.hpo_chunk() == orc.CHUNK, "C and numpy oracles disagree on CHUNK"
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data if a is not None else None


def threads() -> int:
    return int(lib().hpo_set_threads(0))


def sort_dedup_route(ids, vals, total_rows, parts, owner, nranks):
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    vals = np.ascontiguousarray(vals, dtype=F32)
    owner = np.ascontiguousarray(owner, dtype=np.int32)
    T, D = vals.shape
    send_ids = np.empty(T, np.int64)
    send_rows = np.empty((T, D), F32)
    counts = np.empty(T, np.int32)
    inv = np.empty(T, np.int32)
    dest = np.empty(nranks, np.int32)
    U = lib().hpo_sort_dedup_route(_p(ids), _p(vals), T, D, total_rows, parts, _p(owner), nranks,
                                   _p(send_ids), _p(send_rows), _p(counts), _p(inv), _p(dest))
    return {"send_ids": send_ids[:U], "send_rows": send_rows[:U], "counts": counts[:U],
            "inv": inv, "dest_counts": dest, "n_uniq": int(U)}


_KIND = {"sgd": 0, "adagrad": 1, "adam": 2}


def merge_apply(opt, state, ids, rows, hp, step, scale):
    """Group ``ids`` (source order), tree-sum, scale, apply ``opt`` in place."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    rows = np.ascontiguousarray(rows, dtype=F32)
    b1, b2 = hp.get("beta1", 0.9), hp.get("beta2", 0.999)
    s0 = state.get("acc", state.get("m"))
    s1 = state.get("v")
    lr_t = float(orc.adam_lr_t(hp["lr"], b1, b2, step)) if opt == "adam" else 0.0
    for a in (state["w"], s0, s1):
        assert a is None or (a.flags.c_contiguous and a.dtype == F32)
    return lib().hpo_merge_apply(_p(ids), _p(rows), len(ids), rows.shape[1], _KIND[opt],
                                 _p(state["w"]), _p(s0), _p(s1), float(scale), float(F32(hp["lr"])),
                                 float(F32(b1)), float(F32(b2)), float(F32(1.0 - b1)),
                                 float(F32(1.0 - b2)), float(F32(hp.get("eps", 1e-8))), lr_t)


def gather(w, ids):
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    out = np.empty((len(ids), w.shape[1]), F32)
    lib().hpo_gather(_p(w), w.shape[0], _p(ids), len(ids), w.shape[1], _p(out))
    return out


def sparse_step(state, opt, hp, step, batches, total_rows, parts, owner, aggregation="mean"):
    """:func:`oracle.oracle.sparse_step` on the C restatement."""
    n = len(batches)
    sent = [sort_dedup_route(ids, vals, total_rows, parts, owner, n) for ids, vals in batches]
    scale = F32(1.0 / n) if aggregation == "mean" else F32(1.0)
    for o in range(n):
        got_ids, got_rows = [], []
        for s in range(n):
            off = int(sent[s]["dest_counts"][:o].sum())
            cnt = int(sent[s]["dest_counts"][o])
            got_ids.append(sent[s]["send_ids"][off:off + cnt])
            got_rows.append(sent[s]["send_rows"][off:off + cnt])
        ids_o = np.concatenate(got_ids)
        if len(ids_o):
            merge_apply(opt, state, ids_o, np.concatenate(got_rows), hp, step, scale)
    for r, (ids, _) in enumerate(batches):
        sent[r]["out"] = gather(state["w"], ids)
    return sent


def dense_mean(grads, scale):
    """fp32 sum in rank order times scale (bench CPU baseline; the tolerance
    reference stays :func:`oracle.oracle.dense_allreduce`)."""
    gs = [np.ascontiguousarray(g, dtype=F32).reshape(-1) for g in grads]
    ptrs = (C.c_void_p * len(gs))(*[g.ctypes.data for g in gs])
    out = np.empty(gs[0].size, F32)
    lib().hpo_dense_mean(ptrs, len(gs), gs[0].size, float(scale), _p(out))
    return out
