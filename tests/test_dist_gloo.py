"""World-size-2/3 CPU (gloo) run of the hybrid step's host protocol.

Each rank dedups/routes its own batch (oracle K1+K2), exchanges counts and
(id, row) blocks with torch.distributed all_to_all over gloo using the same
layout helpers the CUDA runner uses (`protocol.py`), merges + applies on the
partitions it homes, pulls the updated rows back and stitches them. The result
must equal the single-process oracle step for all ranks (bit-exact)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc
from paper_1808_02621_b200.protocol import offsets, slab_layout

V, D, P, T = 3000, 8, 6, 700
OPT, HP = "adagrad", {"lr": 0.1}


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _batch(rank, step):
    rng = np.random.default_rng(step * 100 + rank)
    ids = (rng.integers(0, V, T) ** 2 % V).astype(np.int64)
    return ids, rng.standard_normal((T, D), dtype=np.float32)


def _a2a(send: np.ndarray, send_counts, recv_counts, n):
    """all-to-all-v of row blocks (dest-major) -> blocks concatenated by source."""
    ro = offsets(recv_counts)
    inp = torch.from_numpy(np.ascontiguousarray(send))
    out = torch.empty((int(ro[-1]),) + send.shape[1:], dtype=inp.dtype)
    dist.all_to_all_single(out, inp, [int(c) for c in recv_counts], [int(c) for c in send_counts])
    return out.numpy()


def _worker(rank, n, port, steps, q):
    try:
        _run(rank, n, port, steps, q)
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, repr(exc)))


def _run(rank, n, port, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=n)
    owner = orc.owner_table("embedding", P, n)
    bounds = orc.partition_bounds(V, P)
    owned, base, rows = slab_layout(bounds, owner, rank)
    full = orc.init_state(OPT, V, D, seed=4)
    slab = {k: np.concatenate([v[bounds[p]:bounds[p + 1]] for p in owned]) for k, v in full.items()}
    ok = True
    for step in range(1, steps + 1):
        ids, vals = _batch(rank, step)
        k1 = orc.sort_dedup_route(ids, vals, V, P, owner, n)
        send_c = k1["dest_counts"]
        recv_t = torch.empty(n, dtype=torch.int32)
        dist.all_to_all_single(recv_t, torch.from_numpy(send_c.astype(np.int32)))
        recv_c = recv_t.numpy()
        r_ids = _a2a(k1["send_ids"], send_c, recv_c, n)
        r_rows = _a2a(k1["send_rows"], send_c, recv_c, n)
        if len(r_ids):
            uniq, sums, _, _ = orc.grouped_tree_sum(r_ids, r_rows)
            p = orc.partition_of(uniq, V, P)
            assert np.all(owner[p] == rank)
            local = base[p] + uniq - bounds[p]
            orc.apply_rows(OPT, slab, local, sums * np.float32(1.0 / n), HP, step)
            p2 = orc.partition_of(r_ids, V, P)
            resp = slab["w"][base[p2] + r_ids - bounds[p2]]
        else:
            resp = np.zeros((0, D), np.float32)
        pulled = _a2a(resp, recv_c, send_c, n)
        out = pulled[k1["inv"]]
        # single-process oracle of the same step for every rank
        orc.sparse_step(full, OPT, HP, step, [_batch(r, step) for r in range(n)], V, P, owner)
        ok &= np.array_equal(out, full["w"][ids])
        for p in owned:
            ok &= np.array_equal(slab["w"][base[p]:base[p] + bounds[p + 1] - bounds[p]],
                                 full["w"][bounds[p]:bounds[p + 1]])
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [2, 3])
def test_gloo_exchange_protocol_matches_oracle(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, n, port, 2, q)) for r in range(n)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(n)}


def test_slab_layout_partitions_table():
    bounds = orc.partition_bounds(1000, 7)
    for n in (1, 2, 3, 8):
        owner = orc.owner_table("softmax", 7, n)
        total = 0
        for r in range(n):
            owned, base, rows = slab_layout(bounds, owner, r)
            assert sorted(owned) == [p for p in range(7) if owner[p] == r]
            total += rows
            assert all(base[p] == -1 for p in range(7) if p not in owned)
        assert total == 1000
