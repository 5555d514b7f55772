"""n emulated ranks in ONE process on ONE GPU (test harness, not a transport).

The peer-memory protocol (``hp_xchg_*`` sparse exchange, ``hp_dar_*`` dense
exchange) only needs every rank's window address. With one process per GPU the
windows are mapped with cudaIpc; here the n "ranks" are n
:class:`~paper_1808_02621_b200.runner.HybridRunner` objects of one process
sharing one GPU, and :class:`LocalWorld` links their windows by address
(``hp_xchg_set_peer_ptr`` / ``hp_dar_set_peer_ptr``). Every kernel, flag and
wait is the multi-GPU one, so a one-GPU test box exercises the whole exchange
(push epilogue, owner scan/rows, k_applied / k_wait, the dense scatter /
reduce-gather) bit for bit against the oracle. NCCL and NVLS transports cannot
be emulated this way (NCCL needs distinct devices; NVLS a multicast object).

Run each rank's ``step(..., timed=False)`` under its own CUDA stream: the ranks'
waits spin on each other's flags, so the n steps must be in flight together.
Nothing may implicitly synchronise the context while they are: no device
allocation (:meth:`HybridRunner.reserve` sizes every buffer first; step_all
does it) and no lazy module load — run with ``CUDA_MODULE_LOADING=EAGER``
(tests/conftest.py sets it): measured on B200, a lazily loaded kernel's first
launch otherwise stalls the enqueue until the spinning waits time out.
"""

from __future__ import annotations


class LocalWorld:
    def __init__(self, n: int):
        if n < 1:
            raise ValueError("n >= 1")
        self.n = n
        self._seq: dict = {}
        self._groups: dict = {}

    def register(self, kind: str, rank: int, x) -> None:
        """Called by every exchange at creation; the k-th exchange of a kind on
        every rank forms one group (ranks build their runners from the same
        plan, so they create exchanges in the same order). The last member links all."""
        k = self._seq.get((kind, rank), 0)
        self._seq[(kind, rank)] = k + 1
        grp = self._groups.setdefault((kind, k), {})
        if rank in grp:
            raise RuntimeError(f"rank {rank} registered {kind} #{k} twice")
        grp[rank] = x
        if len(grp) == self.n:
            shapes = {o.shape for o in grp.values()}
            if len(shapes) != 1:
                raise ValueError(f"{kind} #{k}: window shapes differ across ranks: {shapes}")
            ptrs = {r: o.window_ptr() for r, o in grp.items()}
            for r, o in grp.items():
                for q, p in ptrs.items():
                    if q != r:
                        o.link_peer(q, p)
            del self._groups[(kind, k)]

    @staticmethod
    def serialize(runner) -> None:
        """Run an emulated rank's step on ONE stream (its tables one after
        another, its next plans after them): every rank then meets the
        exchange's waits in the same order on its own stream, which needs n
        hardware queues only. With the concurrent multi-stream step, n ranks x
        (table, plan, dense) streams outnumber the device's connections and
        streams of different ranks share a queue: one rank's spinning wait then
        blocks another rank's work queued behind it (measured: n >= 3 timed out).
        The split push's side stream goes too, for the same reason."""
        runner.concurrent_tables = False
        runner._short_streams = {}

    def comm(self, rank: int) -> "LocalComm":
        return LocalComm(self, rank)


class LocalComm:
    """The ``comm`` a HybridRunner of an emulated rank gets: no NCCL
    communicator (``ptr`` is None), only the world its exchanges link through."""

    def __init__(self, world: LocalWorld, rank: int):
        self.world, self.rank, self.world_size = world, rank, world.n
        self.ptr = None

    def close(self) -> None:
        pass


def step_all(runners: list, streams: list, batches: list, next_batches: list | None = None,
             upcoming: list | None = None) -> None:
    """One hybrid step of every emulated rank, each on its own stream (the
    ranks' device waits depend on each other, so all are enqueued before any
    is waited for), then a device synchronisation."""
    import torch

    for run, b in zip(runners, batches):  # no allocation while waits spin
        run.reserve(b)
    for r, (run, s) in enumerate(zip(runners, streams)):
        with torch.cuda.stream(s):
            run.step(batches[r], timed=False,
                     next_batch=None if next_batches is None else next_batches[r],
                     upcoming=None if upcoming is None else upcoming[r])
    torch.cuda.synchronize()


def capture_pipelined_all(runners: list, streams: list, batches: list,
                          steps_per_graph: int = 1) -> list:
    """:meth:`HybridRunner.capture_pipelined` for every emulated rank:
    ``batches[rank][r]`` is rank's rotation. The eager warm-up rotation runs for
    all ranks together (step_all), then each rank's graphs are captured.
    Replay graph k of every rank on that rank's stream, all ranks together."""
    import torch

    R = len(batches[0])
    L = runners[0].lookahead
    while L > 1 and R % (L + 1):
        L -= 1
    for run, b in zip(runners, batches):
        run.lookahead = L
        for tab in run.tables.values():
            tab.pending.clear()
        run.prefetch(b[0])
    for r in range(R):
        step_all(runners, streams, [b[r] for b in batches],
                 upcoming=[[b[(r + 1 + i) % R] for i in range(L)] for b in batches])
    torch.cuda.synchronize()
    return [run.capture_pipelined(b, steps_per_graph, warm=False) for run, b in zip(runners, batches)]


def replay_all(graphs: list, streams: list, k: int) -> None:
    import torch

    for g, s in zip(graphs, streams):
        with torch.cuda.stream(s):
            g[k].replay()
    torch.cuda.synchronize()
