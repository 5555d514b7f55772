"""Result records of one device step, shaped like the reference's simulator output.

``IterationStats`` keeps the reference's fields (`simulate.py:71-79`):
``iter_time_us``, ``per_machine_bytes`` (a :class:`TransferReport` of
(egress, ingress) bytes per GPU, `transfer.py:30-77`), ``phase_times`` with the
keys compute / network / intra / update (`simulate.py:369-375`) and ``trace``
of :class:`Message` records tagged (variable, partition, phase). Here every
number is MEASURED: times come from CUDA events around each phase, bytes are
counted from the device-side send/receive counts of the exchange.
"""

from __future__ import annotations

from dataclasses import dataclass, field

Endpoint = tuple  # (machine, device)


@dataclass(frozen=True)
class Message:
    """One tagged transfer (reference `simulate.py:30-55`)."""

    src: tuple
    dst: tuple
    nbytes: int
    variable: str
    partition: int
    phase: str

    @property
    def cross_machine(self) -> bool:
        return self.src[0] != self.dst[0]

    def to_dict(self) -> dict:
        return {"src": list(self.src), "dst": list(self.dst), "bytes": self.nbytes,
                "variable": self.variable, "partition": self.partition, "phase": self.phase}


@dataclass(frozen=True)
class TransferReport:
    """Per-GPU (egress, ingress) bytes for one iteration (reference `transfer.py:30-77`)."""

    per_machine: tuple

    def __post_init__(self) -> None:
        object.__setattr__(self, "per_machine", tuple(tuple(p) for p in self.per_machine))

    @property
    def bottleneck_machine(self) -> int:
        return max(range(len(self.per_machine)), key=lambda i: max(self.per_machine[i]))

    @property
    def bottleneck_bytes(self) -> float:
        return max(max(e, i) for e, i in self.per_machine)

    @property
    def total_bytes(self) -> float:
        return sum(e + i for e, i in self.per_machine)

    def machine_total(self, i: int) -> float:
        return sum(self.per_machine[i])

    def __add__(self, other: "TransferReport") -> "TransferReport":
        if len(self.per_machine) != len(other.per_machine):
            raise ValueError("machine counts differ")
        return TransferReport(tuple((a[0] + b[0], a[1] + b[1])
                                    for a, b in zip(self.per_machine, other.per_machine)))

    def to_rows(self) -> list:
        return [{"machine": i, "egress_bytes": e, "ingress_bytes": g}
                for i, (e, g) in enumerate(self.per_machine)]


@dataclass(frozen=True)
class ComputeProfile:
    """Non-network costs of one iteration (reference `simulate.py:58-68`, same
    fields and validation). On the device the aggregation / partition terms are
    measured, not modelled; ``compute_us_per_gpu`` (the model's forward /
    backward, which this path does not run) is added to measured step times by
    :func:`~paper_1808_02621_b200.tuning.tune` and
    :func:`~paper_1808_02621_b200.runner.simulate_training`."""

    compute_us_per_gpu: float = 0.0
    partition_overhead_us: float = 0.0
    agg_us_per_mb: float = 0.0

    def __post_init__(self) -> None:
        from .model import SpecError

        if min(self.compute_us_per_gpu, self.partition_overhead_us, self.agg_us_per_mb) < 0:
            raise SpecError("compute profile fields must be >= 0")


@dataclass(frozen=True)
class IterationStats:
    """Measured counterpart of the reference's ``IterationStats`` (`simulate.py:71-79`)."""

    iter_time_us: float
    per_machine_bytes: TransferReport
    phase_times: dict
    trace: tuple = ()
    counters: dict = field(default_factory=dict)  # unique rows per table etc.

    def update_events(self) -> list:
        return [m for m in self.trace if m.phase == "update"]
