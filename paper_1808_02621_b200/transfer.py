"""Predicted per-GPU exchange bytes of a plan (reference `transfer.py:80-186`).

The reference's closed-form model: with ``w`` a Weight's gradient payload
(``VariableSpec.payload_bytes``: ceil(alpha * elements) * elem_bytes, a dense
Weight has alpha = 1) and ``n`` machines (here: GPUs of one box, one worker
each):

* dense under AR (ring)      every GPU sends and receives 2 w (n-1)/n;
* sparse under AR (AllGatherv) every GPU sends and receives w (n-1);
* a PS partition of payload w homed on owner o: o serves the pull, w (n-1)
  out, and takes one push per other GPU, w (n-1) in; every other GPU sends
  w and receives w.

:class:`HybridRunner` reports the MEASURED bytes of the same step
(``IterationStats.per_machine_bytes``, counted from the device send/receive
counts, ids included); :func:`transfer_model` is printed beside it
(``bench.py`` at N > 1, ``cli simulate``). The model assumes a uniform touched
fraction per partition, so Zipf-skewed ids (a hot partition 0) make the
measured bytes differ: reported, not asserted.
"""

from __future__ import annotations

from .model import ClusterSpec, GraphSpec, SpecError, partition_variable
from .placement import DistributedPlan, Mechanism
from .stats import TransferReport


def _add(acc: list, rows) -> None:
    for m, (eg, ing) in enumerate(rows):
        acc[m][0] += eg
        acc[m][1] += ing


def payload_transfer(payload: float, mech: Mechanism, n: int, owner: int | None,
                     push_multiplier: int = 1, gather_blocks: int = 1) -> list:
    """[egress, ingress] per machine for one payload (reference `transfer.py:80-126`).

    ``push_multiplier``: pushes per machine without local aggregation (G);
    ``gather_blocks``: AllGatherv blocks per machine (G)."""
    out = [[0.0, 0.0] for _ in range(n)]
    if n == 1:
        return out
    if mech is Mechanism.PS:
        if owner is None or not 0 <= owner < n:
            raise SpecError(f"PS transfer requires an owner machine in [0, {n}), got {owner}")
        for m in range(n):
            if m == owner:
                out[m][0] += payload * (n - 1)
                out[m][1] += payload * (n - 1) * push_multiplier
            else:
                out[m][0] += payload * push_multiplier
                out[m][1] += payload
        return out
    if gather_blocks == 1:
        per_dir = payload * (n - 1)
        return [[per_dir, per_dir] for _ in range(n)]
    remote = n * gather_blocks - gather_blocks
    both = payload * gather_blocks * remote
    return [[both, both] for _ in range(n)]


def transfer_model(graph: GraphSpec, plan: DistributedPlan, cluster: ClusterSpec) -> TransferReport:
    """Predicted per-machine (egress, ingress) bytes of one iteration of ``plan``
    (reference `transfer.py:149-186`)."""
    n, g = cluster.machines, cluster.gpus_per_machine
    acc = [[0.0, 0.0] for _ in range(n)]
    pushes = 1 if plan.local_agg_enabled else g
    for var in graph.variables:
        mech = plan.mech_of[var.name]
        if mech is Mechanism.AR:
            if var.kind == "dense":
                per_dir = 2.0 * var.payload_bytes * (n - 1) / n
                _add(acc, [(per_dir, per_dir)] * n)
            else:
                _add(acc, payload_transfer(var.payload_bytes, mech, n, None, gather_blocks=g))
            continue
        for p, elems in partition_variable(var, plan.partitions_of[var.name]).partitions:
            _add(acc, payload_transfer(var.partition_payload_bytes(elems), mech, n,
                                       plan.owner_of(var.name, p), push_multiplier=pushes))
    return TransferReport(tuple((eg, ing) for eg, ing in acc))
