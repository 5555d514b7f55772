"""Host-side layout of the sharded tables and of the (index, row) exchange.

Pure numpy: shared by :class:`runner.HybridRunner` (device path) and the
multi-process CPU tests (gloo), so the bookkeeping both rely on is one code.

* Slab layout: rank r homes every partition p with ``owner[p] == r``; its slab
  is those partitions' rows concatenated in ascending p, so partition p starts
  at slab row ``part_base[p]`` (-1 where not homed). Reference: PS partitions
  homed per server (`sparseplan/placement.py:165-199`).
* Push: a worker's unique rows are in send order (ascending (owner, id)), so
  the rows for rank o are the contiguous block ``[send_off[o], send_off[o] +
  send_counts[o])``. An owner receives the blocks of every source
  concatenated in source-rank order. Pull returns, along the reverse routes,
  one row per received id, so worker row ``k`` of the pulled buffer is the
  post-update row of its send slot ``k`` (reference push/pull,
  `sparseplan/simulate.py:183-214`).
"""

from __future__ import annotations

import numpy as np


def slab_layout(bounds: np.ndarray, owner: np.ndarray, rank: int):
    """(owned partitions, part_base int64[P], slab rows) of ``rank``."""
    P = len(owner)
    base = np.full(P, -1, dtype=np.int64)
    owned = [p for p in range(P) if int(owner[p]) == rank]
    rows = 0
    for p in owned:
        base[p] = rows
        rows += int(bounds[p + 1] - bounds[p])
    return owned, base, rows


def offsets(counts) -> np.ndarray:
    """Exclusive prefix of per-peer counts (block starts in a dest-major buffer)."""
    c = np.asarray(counts, dtype=np.int64)
    out = np.zeros(len(c) + 1, dtype=np.int64)
    np.cumsum(c, out=out[1:])
    return out


def wire_bytes(send_counts, recv_counts, rank: int, D: int, index_bytes: int = 8):
    """(egress, ingress) bytes of one push + pull, excluding the self block."""
    eg = ing = 0
    for o, (s, r) in enumerate(zip(send_counts, recv_counts)):
        if o == rank:
            continue
        eg += s * (index_bytes + 4 * D) + r * 4 * D
        ing += r * (index_bytes + 4 * D) + s * 4 * D
    return eg, ing
