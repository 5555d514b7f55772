"""HybridRunner: one synchronous hybrid-communication step on real devices.

The device counterpart of the reference's ``simulate_iteration`` /
``simulate_training`` (`sparseplan/simulate.py:326-402`): it consumes an
unchanged :class:`DistributedPlan` (from :func:`transform_hybrid`) and runs

* dense (AR) Weights  -> K7 allreduce fused with the 1/n scale + cast;
* sparse (PS) Weights -> K1+K2 sort/dedup/route, K3 push all-to-all,
  K4 owner merge + scatter-apply, K5 owner gather, K3 pull, K6 stitch.
  With one GPU every partition is local (the reference marks every Weight AR
  at one machine, `placement.py:111`) and the step is the fused local apply
  followed by a gather.

Tables live as row slabs: rank r holds the partitions p with owner[p] == r,
concatenated in ascending p (each partition is a separate view,
:meth:`ShardedTable.partition`). ``step()`` returns an ``IterationStats`` with
measured phase times (CUDA events) and measured exchange bytes.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from ._lib import Slab
from .model import ClusterSpec, GraphSpec, SpecError, VariableSpec, partition_bounds
from .ops import OptimizerConfig, Workspace
from .placement import DistributedPlan, Mechanism, transform_hybrid
from .protocol import slab_layout, wire_bytes
from .stats import IterationStats, Message, TransferReport


class ShardedTable:
    """This rank's partitions of one sparse Weight plus optimizer state."""

    def __init__(self, var: VariableSpec, partitions: int, owner: np.ndarray, rank: int,
                 optimizer: OptimizerConfig, device, seed: int = 0, init_scale: float = 0.05,
                 w_storage=None, plan_slots: int = 3):
        if var.elem_bytes % 16:
            raise SpecError(f"table {var.name!r}: row bytes must be a multiple of 16 (D % 4 == 0)")
        self.var = var
        self.name = var.name
        self.V = var.elements
        self.D = var.elem_bytes // 4
        self.P = partitions
        self.rank = rank
        self.optimizer = optimizer
        self.device = torch.device(device)
        self.owner = np.asarray(owner, dtype=np.int32)
        self.bounds = partition_bounds(self.V, self.P)
        self.owned, base, rows = slab_layout(self.bounds, self.owner, rank)
        self.rows = rows
        self.part_base_host = base
        self.part_base = torch.from_numpy(base).to(self.device)
        self.owner_dev = torch.from_numpy(self.owner).to(self.device)
        if w_storage is not None:  # the slab lives in a peer-readable window
            self.w = w_storage(max(rows, 1))
        else:
            self.w = torch.empty(max(rows, 1), self.D, dtype=torch.float32, device=self.device)
        self.state = [torch.empty_like(self.w) for _ in range(optimizer.n_state)]
        for p in self.owned:
            lo, hi = int(self.bounds[p]), int(self.bounds[p + 1])
            ops.init_rows(self.partition(p), lo, seed, init_scale)
        if optimizer.kind == "adagrad":
            ops.fill(self.state[0], optimizer.init_acc)
        elif optimizer.kind == "adam":
            for s in self.state:
                s.zero_()
        # plan workspaces (HybridRunner.lookahead + 1): the plans of the next
        # steps are built while this one applies; step k's plan lives in slot
        # k % (lookahead + 1)
        self.wss = [Workspace(self.device) for _ in range(max(plan_slots, 2))]
        self.applied = 0        # number of this table's next step
        self.pending: dict = {}  # step number -> (ids tensor, slot, event | None)
        self.step_count = 0

    @property
    def ws(self) -> Workspace:
        return self.wss[0]

    def partition(self, p: int) -> torch.Tensor:
        """Partition p as its own [rows_p, D] array (view into the slab)."""
        b = int(self.part_base_host[p])
        if b < 0:
            raise KeyError(f"partition {p} of {self.name!r} is not homed on rank {self.rank}")
        n = int(self.bounds[p + 1] - self.bounds[p])
        return self.w[b:b + n]

    def slab(self) -> Slab:
        s0 = self.state[0].data_ptr() if self.state else None
        s1 = self.state[1].data_ptr() if len(self.state) > 1 else None
        return Slab(self.w.data_ptr(), s0, s1, self.part_base.data_ptr(), self.V, self.P, self.D)

    def state_dict(self) -> dict:
        out = {"w": self.w[:self.rows]}
        for k, s in zip(("acc",) if self.optimizer.kind == "adagrad" else ("m", "v"), self.state):
            out[k] = s[:self.rows]
        return out


@dataclass
class _Scratch:
    """Grow-only per-table exchange buffers."""

    cap: int = 0
    tensors: dict = field(default_factory=dict)


class HybridRunner:
    """Run hybrid-communication steps for ``plan`` on this process's GPU.

    Parameters mirror the reference planner inputs: ``plan`` / ``graph`` /
    ``cluster`` (a one-box cluster is ``ClusterSpec.b200_box(n)``), plus the
    runtime choices the reference leaves to the framework: the sparse row
    optimizer, ``aggregation`` ('mean' divides by n as Horovod/Parallax
    averaging does, 'sum' does not; `PAPER.md:542`) and the dense output dtype.
    """

    def __init__(self, plan: DistributedPlan, graph: GraphSpec, cluster: ClusterSpec, *,
                 rank: int = 0, world_size: int = 1, comm=None,
                 optimizer: OptimizerConfig | None = None, aggregation: str = "mean",
                 dense_dtype: torch.dtype = torch.float32, device=None, seed: int = 0,
                 exchange: str = "p2p", max_ids: dict | None = None,
                 dense_exchange: str | None = None, dense_split="auto",
                 dense_in_dtype: torch.dtype = torch.float32):
        if aggregation not in ("mean", "sum"):
            raise ValueError("aggregation must be 'mean' or 'sum'")
        if cluster.total_gpus != world_size:
            raise SpecError(f"cluster has {cluster.total_gpus} GPUs but world_size={world_size}")
        if world_size > 1 and cluster.gpus_per_machine != 1:
            raise SpecError("one B200 box is ClusterSpec(machines=n_gpus, gpus_per_machine=1)")
        if world_size > 1 and comm is None:
            raise ValueError("world_size > 1 needs a Comm (Comm.from_torch_distributed())")
        if exchange not in ("p2p", "nccl"):
            raise ValueError("exchange must be 'p2p' (NVLink peer memory) or 'nccl'")
        self.exchange = exchange if world_size > 1 else "local"
        # dense allreduce: peer-memory kernel (deterministic, scale/cast fused) or NCCL.
        # Default K7 transport by measurement: the SM-store peer
        # exchange (bit-exact rank-order sum, scale + cast fused) — at n = 2 equal
        # to NCCL in the full LM1B step (138.6 vs 138.4 us) and faster alone
        # (dense-only step 81.7 vs 106.7 us, r2m2b); from 4 ranks its reduction
        # split keeps the hot sparse partitions' owners out of the reduce/gather
        default_dense = "p2p-sm" if exchange == "p2p" else exchange
        self.dense_exchange = (dense_exchange or default_dense) if world_size > 1 else "local"
        if self.dense_exchange not in ("p2p", "p2p-sm", "p2p-pipe", "p2p-pull", "nvls", "nccl",
                                       "local"):
            raise ValueError("dense_exchange must be 'p2p' (copy engines), 'p2p-sm', "
                             "'p2p-pipe', 'p2p-pull', 'nvls' or 'nccl'")
        self._world = getattr(comm, "world", None)  # emulated ranks (emulate.LocalWorld)
        if self._world is not None and (self.exchange != "p2p" or self.dense_exchange in
                                        ("nccl", "nvls")):
            raise ValueError("emulated ranks (LocalWorld) run the peer-memory transports only: "
                             "exchange='p2p', dense_exchange in ('p2p', 'p2p-sm', 'p2p-pipe', "
                             "'p2p-pull')")
        self.dar: dict = {}
        self.dense_weights = None  # reduction share per rank of the peer dense exchange
        self.xchg: dict = {}
        self.ar_tables: set = set()   # sparse Weights under AR at n > 1 (AllGatherv baseline)
        self.dense_ps: dict = {}      # dense Weights under PS at n > 1: name -> owner rank
        self.glob_base: dict = {}
        self.plan, self.graph, self.cluster = plan, graph, cluster
        self.rank, self.world_size, self.comm = rank, world_size, comm
        self.optimizer = optimizer or OptimizerConfig()
        self.aggregation = aggregation
        self.scale = 1.0 / world_size if aggregation == "mean" else 1.0
        self.dense_dtype = dense_dtype
        # dense gradients arrive in fp32 or bf16 (SURVEY §8b in_dtype): bf16 is
        # widened exactly and summed in fp32; over peer memory it travels as
        # bf16 (SM stores: half the NVLink bytes)
        if dense_in_dtype not in (torch.float32, torch.bfloat16):
            raise ValueError("dense_in_dtype must be torch.float32 or torch.bfloat16")
        if dense_in_dtype == torch.bfloat16 and world_size > 1 and self.dense_exchange not in (
                "p2p-sm", "nccl"):
            raise ValueError("bf16 dense gradients run over dense_exchange 'p2p-sm' or 'nccl'")
        self.dense_in_dtype = dense_in_dtype
        self.device = torch.device(device if device is not None else torch.cuda.current_device())
        self.seed = seed
        self.tables: dict[str, ShardedTable] = {}
        self.dense: list[VariableSpec] = []
        for i, var in enumerate(graph.variables):
            mech = plan.mech_of[var.name]
            if var.kind == "dense":
                self.dense.append(var)
                if mech is Mechanism.PS and world_size > 1:  # reduce at the owner + broadcast
                    if dense_in_dtype != torch.float32:
                        raise ValueError("a dense Weight under PS takes fp32 gradients")
                    self.dense_ps[var.name] = plan.owner_of(var.name, 0)
                elif self.dense_exchange == "nvls":
                    from .xchg import NvlsExchange

                    self.dar[var.name] = NvlsExchange(world_size, rank, var.elements,
                                                      dense_dtype, self.device)
                elif self.dense_exchange in ("p2p", "p2p-sm", "p2p-pipe", "p2p-pull"):
                    from .xchg import DenseExchange

                    self.dar[var.name] = DenseExchange(
                        world_size, rank, var.elements, dense_dtype, self.device,
                        mode={"p2p": "ce", "p2p-sm": "sm", "p2p-pipe": "pipe",
                              "p2p-pull": "pull"}[self.dense_exchange],
                        world=self._world, in_dtype=dense_in_dtype)
                    w = self._dense_split_weights(dense_split)
                    if w is not None:
                        self.dar[var.name].set_split(w)
                    self.dense_weights = w
                continue
            if mech is Mechanism.PS:
                P = plan.partitions_of[var.name]
                owner = plan.owner_table(var.name)
            elif world_size == 1:
                P, owner = 1, np.zeros(1, dtype=np.int32)  # AR over one replica: local apply
            else:  # AR at n > 1: a full replica per rank, fed by an AllGatherv of the slices
                P, owner = 1, np.array([rank], dtype=np.int32)
                self.ar_tables.add(var.name)
            storage = None
            if self.exchange == "p2p" and var.name not in self.ar_tables:
                storage = self._make_window(var, P, owner, (max_ids or {}).get(var.name))
            self.tables[var.name] = ShardedTable(var, P, owner, rank, self.optimizer,
                                                 self.device, seed=seed * 1000 + i,
                                                 w_storage=storage, plan_slots=3)
        self._scratch: dict[str, _Scratch] = {n: _Scratch() for n in self.tables}
        if self.optimizer.kind == "adam":  # step size read on the device: graph-safe
            steps = np.arange(1 << 16, dtype=np.float64)
            steps[0] = 1.0
            self._lr_t_table = torch.from_numpy(self.optimizer.lr_t(steps)).to(self.device)
            for tab in self.tables.values():
                tab.step_dev = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.dense_out: dict[str, torch.Tensor] = {}
        self._dense_bufs: dict[str, dict] = {}
        self.outputs: dict[str, torch.Tensor] = {}
        self.step_count = 0
        self.last_counts: dict = {}
        self.kernel_events: dict | None = None
        # Stream priorities (lower = scheduled first; measured). One
        # GPU: the next step's plans (latency-bound cluster sort) first, then the
        # tables' apply chains, the dense scale/cast last. Several GPUs: the dense
        # exchange (NVLink-bound, on the step's critical path) with the plans,
        # ahead of the tables. HP_STREAM_PRIO="table,dense,plan" overrides.
        default_prio = "-1,0,-2" if world_size == 1 else "-1,-2,-2"
        prio = [int(x) for x in os.environ.get("HP_STREAM_PRIO", default_prio).split(",")]
        pt, pd, pp = prio[:3]
        pbig = prio[3] if len(prio) > 3 else pt  # optional: the largest table's chain
        big = max(self.tables.values(), default=None,  # most rows touched per step
                  key=lambda t: graph.variable(t.name).touched_elements * t.D)
        self._streams = {n: torch.cuda.Stream(device=self.device,
                                              priority=pbig if big is not None and n == big.name
                                              else pt)
                         for n in self.tables}
        self._dense_stream = torch.cuda.Stream(device=self.device, priority=pd)
        # each table's short segments (n = 1: reduce + apply + pull,
        # hp_apply_plan_pull; n > 1: reduce + peer stores, hp_xchg_push_plan)
        # run on a side stream beside its long segments' chain; one priority
        # step below the chain. Default at n = 1 (HP_SPLIT_LONG=0: one stream);
        # at n > 1 only with HP_SPLIT_PUSH=1 (measured neutral at N = 2: full
        # step 134.0 vs 136.6 us, sparse-only 96.6 vs 92.9 us, the push alone
        # 42 vs 38 us)
        split = (os.environ.get("HP_SPLIT_LONG", "1") == "1" if world_size == 1
                 else os.environ.get("HP_SPLIT_PUSH", "0") == "1")
        self._short_streams = ({n: torch.cuda.Stream(device=self.device, priority=min(pt + 1, 0))
                                for n in self.tables} if split else {})
        # two plan streams per table, alternating by step: the dedup of step s+1
        # may start before the one of step s has finished (each is a latency-
        # bound cluster sort on a few SMs, about as long as a whole step)
        self._plan_streams = {n: [torch.cuda.Stream(device=self.device, priority=pp)
                                  for _ in range(2)]
                              for n in self.tables}
        self._pending_counts: dict = {}
        self._ps_used: set = set()  # plan streams forked since the last join
        self._want_counts = False
        # NVTX ranges around the step and its phases (HP_NVTX=1; ncu --nvtx filters)
        self.nvtx = os.environ.get("HP_NVTX", "0") == "1"
        self.concurrent_tables = True
        # Plans built ahead (pipelined steps): with lookahead L the dedup of step
        # k + L runs on the plan streams during step k, so a step never waits for
        # the next plan (the latency-bound cluster sort, ~28 us at LM1B shapes,
        # was the N=1 step's critical path with L = 1). Slots: L + 1 <= 3.
        self.lookahead = min(max(int(os.environ.get("HP_LOOKAHEAD", "2")), 1), 2)
        # captured steps run with per-node priorities (ops.StepGraph)
        self.graph_node_priority = os.environ.get("HP_GRAPH_NODE_PRIORITY", "1") != "0"
        # device error bits -> pinned host words (one per table stream + dense),
        # collected on the streams that own them, read at the next step()
        self._err = ops.ErrorWords(len(self.tables) + 1)
        self._err_slot = {n: i for i, n in enumerate(self.tables)}

    def _dense_split_weights(self, dense_split):
        """Reduction share per rank for the peer-memory dense exchange.

        'auto': with frequency-ranked row ids (LM vocabularies, the Zipf inputs of
        BASELINE's configs) partition 0 of a sparse Weight is its hot range, so
        the rank homing it carries most of that Weight's push/return NVLink
        traffic. 'auto' gives those ranks no dense reduction
        chunk (weight 0) when n >= 4 and at least one rank stays. 'uniform', or
        an explicit list of n weights, overrides it. The pipelined transport
        keeps the uniform split."""
        n = self.world_size
        if isinstance(dense_split, (list, tuple)):
            if len(dense_split) != n:
                raise ValueError(f"dense_split needs {n} weights")
            return list(dense_split)
        if dense_split in (None, "uniform") or self.dense_exchange in ("p2p-pipe", "p2p-pull") or n < 4:
            return None
        if dense_split != "auto":
            raise ValueError("dense_split: 'auto', 'uniform' or a list of weights")
        hot = {self.plan.owner_of(v.name, 0) for v in self.graph.variables
               if v.kind == "sparse" and self.plan.mech_of[v.name] is Mechanism.PS}
        if not hot or len(hot) >= n:
            return None
        return [0.0 if r in hot else 1.0 for r in range(n)]

    def _make_window(self, var: VariableSpec, P: int, owner: np.ndarray, max_ids):
        """Create the table's peer window; returns the slab allocator for ShardedTable.

        Inbox capacity per source = the most unique rows one worker can send to
        one owner: bounded by the ids per worker per step, i.e. the Weight's
        touched rows ceil(alpha * V) (reference `model.py:27-33,73-81`) unless
        ``max_ids`` overrides it.
        """
        from .xchg import PeerExchange

        D = var.elem_bytes // 4
        bounds = partition_bounds(var.elements, P)
        cap = int(max_ids or var.touched_elements)
        # the window layout must be identical on every rank (peers address each
        # other's inboxes with their own offsets): size the slab region for the
        # largest slab of any rank (P not a multiple of n gives unequal slabs)
        rows_cap = max(max(slab_layout(bounds, owner, r)[2] for r in range(self.world_size)), 1)
        x = PeerExchange(self.world_size, self.rank, D, cap, rows_cap, self.device,
                         world=self._world)
        self.xchg[var.name] = x
        gb = np.zeros(P, dtype=np.int64)
        for r in range(self.world_size):
            _, base, _ = slab_layout(bounds, owner, r)
            gb[base >= 0] = base[base >= 0]
        self.glob_base[var.name] = torch.from_numpy(gb).to(self.device)
        return lambda nrows: x.w[:nrows]

    def _sparse_p2p(self, tab: ShardedTable, ids, vals, opt, slot: int = 0,
                    planned: bool = False) -> torch.Tensor:
        n, D, T = self.world_size, tab.D, ids.numel()
        name = tab.name
        x = self.xchg[name]
        if T > x.cap:
            raise SpecError(f"table {name!r}: {T} ids exceed the inbox capacity {x.cap} "
                            "(raise max_ids)")
        k = self._kev
        r = self._p2p_bufs(tab, slot)
        if not planned:
            self._plan(tab, ids, slot)
        k(f"push:{name}", True)
        x.push_plan(vals, tab.V, tab.P, r, self.glob_base[name], tab.wss[slot],
                    side_stream=self._short_streams.get(name))
        k(f"push:{name}", False)
        # Waits stay one-block kernels (k_wait): folded into the prologue of the
        # owner scan / stitch, every block of those grids spun, holding SMs the
        # other tables' concurrent chains need (and deadlocking the one-GPU
        # emulation of 4 ranks, whose waits then outnumber the SM slots)
        k(f"wait_push:{name}", True)
        x.wait(0)
        k(f"wait_push:{name}", False)
        k(f"apply:{name}", True)
        x.merge_apply(tab.slab(), opt, wait=False)
        k(f"apply:{name}", False)
        if self._want_counts:  # exchange bytes of a timed step (a memcpy off the graphs)
            rc = self._buf(name, "recv_counts", (n,), torch.int32)
            x.recv_counts(rc)
            self._pending_counts[name] = (r["dest_counts"], rc)
        out = self._buf(name, "out", (T, D), torch.float32)
        k(f"wait_applied:{name}", True)
        x.wait(1)
        k(f"wait_applied:{name}", False)
        k(f"stitch:{name}", True)
        x.stitch_plan(tab.wss[slot], T, tab.V, tab.P, out, wait=False)
        k(f"stitch:{name}", False)
        return out

    def exchange_status(self) -> dict:
        """Error bits of every peer exchange, sparse and dense (synchronises)."""
        out = {k: x.status() for k, x in self.xchg.items()}
        out.update({f"dense:{k}": d.status() for k, d in self.dar.items()})
        return out

    def close(self) -> None:
        for x in list(self.xchg.values()) + list(self.dar.values()):
            x.close()
        self.xchg.clear()
        self.dar.clear()
        if self._err is not None:
            torch.cuda.synchronize(self.device)
            self._err.close()
            self._err = None

    # ------------------------------------------------------------------ step
    def _buf(self, name: str, key: str, shape, dtype) -> torch.Tensor:
        sc = self._scratch[name]
        t = sc.tensors.get(key)
        numel = int(np.prod(shape))
        if t is None or t.numel() < numel or t.dtype != dtype:
            t = torch.empty(max(numel, 1), dtype=dtype, device=self.device)
            sc.tensors[key] = t
        return t[:numel].view(*shape) if len(shape) > 0 else t

    def _kev(self, key: str, begin: bool) -> None:
        """Per-kernel CUDA events (bench roofline); off unless kernel_events is a dict."""
        if self.kernel_events is None:
            return
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream())
        self.kernel_events.setdefault(key, []).append(e)

    # bit layout of the runner's error words
    ERR_BITS = {1: "an id outside [0, V) was dropped (no row updated, zero row pulled)",
                2: "a row id is not homed on this rank",
                4: "a sparse push wait timed out (the owner merged nothing)",
                8: "a sparse apply wait timed out (pulled rows are stale)",
                16: "a received row id is not homed on its owner",
                4 << 8: "a dense-exchange scatter wait timed out",
                8 << 8: "a dense-exchange gather wait timed out"}

    def _collect_errors(self, tab: ShardedTable, slot: int) -> None:
        """Enqueue (current stream) the error words of plan slot ``slot`` and of
        the table's exchange into the table's host word."""
        src = [(ops.plan_err_ptr(tab.wss[slot]), 0)]
        if tab.name in self.xchg:
            src.append((self.xchg[tab.name].err_ptr(), 0))
        self._err.collect(self._err_slot[tab.name], src)

    def _collect_dense_errors(self) -> None:
        src = [(d.err_ptr(), 8) for d in self.dar.values()]
        self._err.collect(len(self.tables), src)

    def check_errors(self, sync: bool = False) -> None:
        """Raise :class:`HybridPathError` if any device error bit reached the host.

        ``step()`` calls this first (no synchronisation), so a failure in step i
        raises from step i+1 at the latest one step after it completed.
        ``sync=True`` collects every word now and waits for the GPU (end of a
        run, or after graph replays)."""
        from ._lib import HybridPathError

        if self.comm is not None and getattr(self.comm, "ptr", None) and hasattr(self.comm, "status"):
            rc = self.comm.status()  # NCCL asynchronous error (host-only poll)
            if rc not in (0, 7):     # ncclSuccess, ncclInProgress
                raise HybridPathError(f"rank {self.rank}: NCCL asynchronous error {rc}")
        if sync:
            for tab in self.tables.values():
                for slot in (0, 1):
                    self._collect_errors(tab, slot)
            self._collect_dense_errors()
            torch.cuda.synchronize(self.device)
        words = self._err.read()
        if not any(words):
            return
        self._err.clear()
        names = list(self.tables) + ["dense"]
        msgs = [f"{names[i]}: {text}" for i, w in enumerate(words) for bit, text in
                self.ERR_BITS.items() if w & bit]
        raise HybridPathError(f"rank {self.rank}: device error bits {words}: " + "; ".join(msgs))

    def _plan(self, tab: ShardedTable, ids, slot: int) -> None:
        """Index half of the step (dedup + route) into plan slot ``slot``, then
        its error word (a dropped id is known as soon as the plan exists) and the
        table's sticky exchange word (the steps before) go to the host word."""
        if self.world_size == 1:
            ops.apply_plan_build(ids, tab.slab(), tab.wss[slot])
        else:
            self.xchg[tab.name].plan(ids, tab.V, tab.P, tab.owner_dev, self.glob_base[tab.name],
                                     self._p2p_bufs(tab, slot), tab.wss[slot])
        self._collect_errors(tab, slot)

    def _p2p_bufs(self, tab: ShardedTable, slot: int) -> dict:
        bufs = self._scratch[tab.name].tensors
        key = f"p2p{slot}"
        if key not in bufs:
            cap, n = self.xchg[tab.name].cap, self.world_size
            bufs[key] = {"send_ids": torch.empty(cap, dtype=torch.int64, device=self.device),
                         "inv": torch.empty(cap, dtype=torch.int32, device=self.device),
                         "dest_counts": torch.empty(n, dtype=torch.int32, device=self.device),
                         "n_uniq": torch.empty(1, dtype=torch.int32, device=self.device)}
        return bufs[key]

    def _sparse_local(self, tab: ShardedTable, ids, vals, opt, slot: int = 0,
                      planned: bool = False) -> torch.Tensor:
        T = ids.numel()
        slab = tab.slab()
        if not planned:
            self._plan(tab, ids, slot)
        out = self._buf(tab.name, "out", (T, tab.D), torch.float32)
        self._kev(f"k4:{tab.name}", True)  # K4 + K5: apply, and the pull fused into it
        ops.apply_plan_pull(vals, T, slab, opt, out, tab.wss[slot],
                            side_stream=self._short_streams.get(tab.name))
        self._kev(f"k4:{tab.name}", False)
        return out

    def _sparse_ar(self, tab: ShardedTable, ids, vals, opt) -> torch.Tensor:
        """A sparse Weight under AR (SURVEY §8f baseline; reference AllGatherv,
        `simulate.py:138-180`): every rank gathers every rank's raw slices and
        applies the concatenation to its own full replica (same result on all
        ranks), then pulls its rows locally. T must be equal on all ranks."""
        n, T, D = self.world_size, ids.numel(), tab.D
        comm = self.comm.ptr
        ids_all = self._buf(tab.name, "ar_ids", (n * T,), torch.int64)
        vals_all = self._buf(tab.name, "ar_vals", (n * T, D), torch.float32)
        ops.allgather(comm, ids.contiguous(), ids_all)
        ops.allgather(comm, vals.contiguous(), vals_all)
        slab = tab.slab()
        ops.apply_plan_build(ids_all, slab, tab.wss[0])
        self._collect_errors(tab, 0)
        self._kev(f"k4:{tab.name}", True)
        ops.apply_plan(vals_all, n * T, slab, opt, tab.wss[0])
        self._kev(f"k4:{tab.name}", False)
        out = self._buf(tab.name, "out", (T, D), torch.float32)
        ops.gather_rows(slab, ids, out)
        return out

    def _sparse_exchange(self, tab: ShardedTable, ids, vals, opt, ev) -> torch.Tensor:
        n, D, T = self.world_size, tab.D, ids.numel()
        name = tab.name
        r = ops.sort_dedup_route(ids, vals, tab.V, tab.P, tab.owner_dev, n, tab.ws,
                                 out=self._scratch[name].tensors.setdefault("k1", {}))
        self._collect_errors(tab, 0)
        recv_counts = self._buf(name, "recv_counts", (n,), torch.int32)
        self.comm.alltoall_counts(r["dest_counts"], recv_counts)
        both = torch.cat([r["dest_counts"], recv_counts]).cpu()  # host counts for NCCL a2a-v
        send_c = both[:n].tolist()
        recv_c = both[n:].tolist()
        R = int(sum(recv_c))
        ev("intra")
        recv_ids = self._buf(name, "recv_ids", (max(R, 1),), torch.int64)
        recv_rows = self._buf(name, "recv_rows", (max(R, 1), D), torch.float32)
        self.comm.push(r["send_ids"], r["send_rows"], send_c, recv_ids, recv_rows, recv_c, D)
        ev("network")
        ops.merge_apply(recv_ids, recv_rows, R, tab.slab(), opt, tab.ws)
        resp = self._buf(name, "resp", (max(R, 1), D), torch.float32)
        ops.gather_rows(tab.slab(), recv_ids, resp, n=R)
        ev("update")
        pulled = self._buf(name, "pulled", (max(int(sum(send_c)), 1), D), torch.float32)
        self.comm.pull(resp, recv_c, pulled, send_c, D)
        ev("network")
        out = self._buf(name, "out", (T, D), torch.float32)
        ops.stitch(pulled, r["inv"], out)
        ev("update")
        self.last_counts[name] = {"send": send_c, "recv": recv_c}
        return out

    def step(self, batch: dict, timed: bool = True, next_batch: dict | None = None,
             upcoming: list | None = None) -> IterationStats:
        """One synchronous hybrid step.

        ``batch[name]`` is ``(ids int64[T], vals f32[T, D])`` for a sparse Weight
        and an fp32 gradient tensor for a dense one (all on this GPU). Pulled
        rows land in ``self.outputs[name]``; averaged dense gradients in
        ``self.dense_out[name]``.

        ``next_batch`` (optional): the batch of the following step, or
        ``upcoming``: the batches of the following steps, in order. Their dedup
        / routing plans (which depend only on their ids) are built on the plan
        streams while this step applies, up to ``lookahead`` steps ahead, each
        into its own plan slot; those steps then skip their dedup. Results are
        identical.
        """
        ahead = list(upcoming) if upcoming is not None else (
            [next_batch] if next_batch is not None else [])
        self.check_errors()
        self._want_counts = timed
        self._pending_counts = {}
        self.step_count += 1
        if self.nvtx:
            torch.cuda.nvtx.range_push(f"hp.step {self.step_count}")
        stream = torch.cuda.current_stream()
        phases = {"compute": 0.0, "network": 0.0, "intra": 0.0, "update": 0.0}
        marks = []

        def ev(phase):
            if timed:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                marks.append((phase, e))

        ev("start")
        t0 = time.perf_counter()
        # NCCL calls of one communicator must not run on concurrent streams: the
        # AR-sparse / PS-dense baselines (NCCL on the table streams) run serially
        concurrent = self.concurrent_tables and (
            self.world_size == 1 or (self.exchange == "p2p" and not self.ar_tables
                                     and not self.dense_ps))
        if concurrent:
            # The dense allreduce and every table are independent: each runs on
            # its own stream (parallel branches when captured as a CUDA graph).
            # The reference serialises these phases; overlap
            # is its named extension point.
            joins = []
            # Plans of the upcoming steps first (enqueue order = node order in a
            # captured graph; the cluster dedup is latency-bound). Each is
            # waited for by the step that applies it (an event), not joined here.
            self._plan_ahead(ahead, stream)
            if self.dense:
                self._dense_stream.wait_stream(stream)
                with torch.cuda.stream(self._dense_stream):
                    self._collect_dense_errors()  # the previous step's (sticky) words
                    self._dense(batch)
                joins.append(self._dense_stream)
            for name, tab in self.tables.items():
                side = self._streams[name]
                side.wait_stream(stream)
                slot, planned, evt = self._take_plan(tab, batch[name][0])
                if evt is not None:
                    side.wait_event(evt)
                with torch.cuda.stream(side):
                    self.outputs[name] = self._sparse(tab, batch[name], None, slot, planned)
                joins.append(side)
            for side in joins:
                stream.wait_stream(side)
            ev("network" if self.world_size > 1 else "update")
        else:
            if self.dense:
                self._collect_dense_errors()
                self._dense(batch)
                ev("network")
            for name, tab in self.tables.items():
                slot, planned, _ = self._take_plan(tab, batch[name][0])
                self.outputs[name] = self._sparse(tab, batch[name], ev, slot, planned)
            self._plan_ahead(ahead, None)  # same stream, after the tables
        if self.nvtx:
            torch.cuda.nvtx.range_pop()
        if timed:
            stream.synchronize()
            for name, (sc, rc) in self._pending_counts.items():
                self.last_counts[name] = {"send": sc.tolist(), "recv": rc.tolist()}
            for (_, a), (ph, b) in zip(marks, marks[1:]):
                phases[ph] += a.elapsed_time(b) * 1e3
            iter_us = marks[0][1].elapsed_time(marks[-1][1]) * 1e3
        else:
            iter_us = (time.perf_counter() - t0) * 1e6
        return IterationStats(iter_us, self._bytes_report(), phases, self._trace(),
                              {"step": self.step_count})

    def _dense_buf(self, var: VariableSpec, key: str, shape, dtype) -> torch.Tensor:
        """Runner-owned persistent buffer of one dense Weight (never a caller tensor)."""
        bufs = self._dense_bufs.setdefault(var.name, {})
        t = bufs.get(key)
        if t is None or tuple(t.shape) != tuple(shape) or t.dtype != dtype:
            t = torch.empty(shape, dtype=dtype, device=self.device)
            bufs[key] = t
        return t

    def dense_is_noop(self) -> bool:
        """K7 does no work at all: one replica, fp32 output, scale 1 ('mean' over
        one rank): the averaged gradient IS this step's gradient."""
        return (self.world_size == 1 and self.dense_dtype == torch.float32
                and self.dense_in_dtype == torch.float32
                and np.float32(self.scale) == np.float32(1.0))

    def _dense(self, batch: dict) -> None:
        if self.nvtx:
            torch.cuda.nvtx.range_push("hp.dense")
        try:
            self._dense_body(batch)
        finally:
            if self.nvtx:
                torch.cuda.nvtx.range_pop()

    def _dense_body(self, batch: dict) -> None:
        """K7 for every dense Weight. The result lands in ``dense_out[name]``:
        a runner-owned buffer (or the exchange window), so the caller's gradient
        tensors are only read; at n=1 with fp32 and scale 1 nothing is launched
        and ``dense_out[name]`` is this step's gradient itself."""
        for var in self.dense:
            g = batch[var.name]
            ops._need(g, self.dense_in_dtype, f"dense gradient {var.name!r}")
            if g.numel() != var.elements:
                raise SpecError(f"dense Weight {var.name!r}: gradient has {g.numel()} elements, "
                                f"the graph declares {var.elements}")
            if self.dense_is_noop():
                self.dense_out[var.name] = g
                continue
            self._kev(f"k7:{var.name}", True)
            if var.name in self.dar:
                self.dense_out[var.name] = self.dar[var.name].allreduce(g, self.scale)
            elif var.name in self.dense_ps:
                out = self._dense_buf(var, "out", (g.numel(),), self.dense_dtype).view(g.shape)
                src = g
                if self.dense_dtype != torch.float32:  # the owner reduces into its input
                    src = self._dense_buf(var, "red", (g.numel(),), torch.float32).view(g.shape)
                    src.copy_(g)
                self.dense_out[var.name] = ops.dense_reduce_bcast(
                    self.comm.ptr, src, out, self.scale, self.dense_ps[var.name])
            elif self.dense_in_dtype != torch.float32:  # bf16 in: widened into fp32 scratch
                out = self._dense_buf(var, "out", (g.numel(),), self.dense_dtype).view(g.shape)
                comm = self.comm.ptr if self.comm is not None else None
                red = (self._dense_buf(var, "red", (g.numel(),), torch.float32)
                       if self.world_size > 1 else None)
                ops.dense_allreduce_scale_cast(comm, g, out, self.scale, scratch=red)
                self.dense_out[var.name] = out
            else:
                out = self._dense_buf(var, "out", (g.numel(),), self.dense_dtype).view(g.shape)
                comm = self.comm.ptr if self.comm is not None else None
                if self.world_size > 1 and self.dense_dtype != torch.float32:
                    # NCCL reduces fp32 with the scale folded in (PreMulSum) into a
                    # runner buffer; the cast then runs as its own epilogue
                    red = self._dense_buf(var, "red", (g.numel(),), torch.float32).view(g.shape)
                    ops.dense_allreduce_scale_cast(comm, g, red, self.scale)
                    ops.dense_allreduce_scale_cast(None, red, out, 1.0)
                else:
                    ops.dense_allreduce_scale_cast(comm, g, out, self.scale)
                self.dense_out[var.name] = out
            self._kev(f"k7:{var.name}", False)

    def _sparse(self, tab: ShardedTable, ids_vals, ev=None, slot: int = 0,
                planned: bool = False) -> torch.Tensor:
        if self.nvtx:
            torch.cuda.nvtx.range_push(f"hp.sparse {tab.name}")
        try:
            return self._sparse_body(tab, ids_vals, ev, slot, planned)
        finally:
            if self.nvtx:
                torch.cuda.nvtx.range_pop()

    def _sparse_body(self, tab: ShardedTable, ids_vals, ev, slot: int, planned: bool) -> torch.Tensor:
        ids, vals = ids_vals
        tab.step_count += 1
        if self.optimizer.kind == "adam":
            ops.step_counter_inc(tab.step_dev)
            opt = self.optimizer.c_struct(tab.step_count, self.scale, self._lr_t_table,
                                          tab.step_dev)
        else:
            opt = self.optimizer.c_struct(tab.step_count, self.scale)
        if self.world_size == 1:
            out = self._sparse_local(tab, ids, vals, opt, slot, planned)
            if ev:
                ev("update")
        elif tab.name in self.ar_tables:
            out = self._sparse_ar(tab, ids, vals, opt)
            if ev:
                ev("network")
        elif self.exchange == "p2p":
            out = self._sparse_p2p(tab, ids, vals, opt, slot, planned)
            if ev:
                ev("network")
        else:
            out = self._sparse_exchange(tab, ids, vals, opt, ev or (lambda _p: None))
        return out

    def pull(self, name: str, ids: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Forward lookup of a sparse Weight: out[t] = its current row ids[t]
        (zero row for an id outside [0, V)), on the current stream.

        One GPU (or a replicated AR table): a local gather. Several GPUs (p2p
        exchange): each row is read straight from its owner's slab over NVLink
        (``hp_xchg_pull``); call it between steps — after the previous step's
        stitch has waited for every owner, before the next step's push."""
        tab = self.tables[name]
        ops._need(ids, torch.int64, "ids", 1)
        if out is None:
            out = torch.empty(ids.numel(), tab.D, dtype=torch.float32, device=self.device)
        ops._need(out, torch.float32, "out", 2)
        if out.shape[0] < ids.numel() or out.shape[1] != tab.D:
            raise ValueError(f"out must be at least [{ids.numel()}, {tab.D}]")
        if self.world_size == 1 or name in self.ar_tables:
            return ops.gather_rows(tab.slab(), ids, out)
        if name not in self.xchg:
            raise NotImplementedError("the forward pull reads owners' slabs over peer memory "
                                      "(exchange='p2p')")
        self.xchg[name].pull(ids, tab.V, tab.P, tab.owner_dev, self.glob_base[name], out)
        return out

    @property
    def plan_slots(self) -> int:
        return self.lookahead + 1

    def _take_plan(self, tab: ShardedTable, ids):
        """(slot, planned, event) of this table's current step; advances its step
        number. A plan built ahead for different ids is discarded."""
        k = tab.applied
        tab.applied += 1
        ent = tab.pending.pop(k, None)
        if ent is not None and ent[0] is ids:
            return ent[1], True, ent[2]
        return k % self.plan_slots, False, None

    def _plan_ahead(self, ahead: list, stream) -> None:
        """Build the plans of the next ``lookahead`` steps that are not built yet,
        on each table's plan stream (``stream`` given: after it, with an event
        for the consumer) or on the current stream (``stream`` None)."""
        if not ahead or not self.pipelined:
            return
        for name, tab in self.tables.items():
            k = tab.applied
            waited = []
            for i, b in enumerate(ahead[:self.lookahead]):
                sn, ids = k + 1 + i, b[name][0]
                ent = tab.pending.get(sn)
                if ent is not None and ent[0] is ids:
                    continue
                slot = sn % self.plan_slots  # last read by step sn - slots < k: done
                if stream is None:
                    self._plan(tab, ids, slot)
                    tab.pending[sn] = (ids, slot, None)
                    continue
                ps = self._plan_streams[name][sn % 2]
                if ps not in waited:
                    ps.wait_stream(stream)
                    waited.append(ps)
                    self._ps_used.add((name, sn % 2))
                with torch.cuda.stream(ps):
                    self._plan(tab, ids, slot)
                e = torch.cuda.Event()
                e.record(ps)
                tab.pending[sn] = (ids, slot, e)

    def _join_plan_streams(self) -> None:
        """The current stream waits for the plan streams used since the last
        join (end of a capture: only streams forked into it may be joined)."""
        cur = torch.cuda.current_stream()
        for name, j in sorted(self._ps_used):
            cur.wait_stream(self._plan_streams[name][j])
        self._ps_used.clear()

    @property
    def pipelined(self) -> bool:
        return ((self.world_size == 1 or self.exchange == "p2p") and not self.ar_tables
                and not self.dense_ps)

    def reserve(self, batch: dict) -> None:
        """Allocate every buffer a step on ``batch``'s shapes uses (both plan
        slots, exchange scratch, outputs) without launching the step. After it,
        steps of these shapes never call the device allocator, which matters
        when several ranks' steps share one GPU (:mod:`.emulate`): an
        allocation is an implicit synchronisation point that would wait on the
        other ranks' spinning exchange waits."""
        n = self.world_size
        for name, tab in self.tables.items():
            T = batch[name][0].numel()
            Tw = T * n if name in self.ar_tables else T
            for ws in tab.wss:
                ws.get(ops.dedup_ws_bytes(Tw, tab.D, tab.P, n))
            self._buf(name, "out", (T, tab.D), torch.float32)
            if name in self.ar_tables:
                self._buf(name, "ar_ids", (n * T,), torch.int64)
                self._buf(name, "ar_vals", (n * T, tab.D), torch.float32)
            elif n > 1 and self.exchange == "p2p":
                for slot in range(len(tab.wss)):
                    self._p2p_bufs(tab, slot)
                self._buf(name, "recv_counts", (n,), torch.int32)
        for var in self.dense:
            if self.dense_is_noop() or var.name in self.dar:
                continue
            self._dense_buf(var, "out", (var.elements,), self.dense_dtype)
            if (self.dense_dtype != torch.float32 or self.dense_in_dtype != torch.float32) and (
                    n > 1 or var.name in self.dense_ps):
                self._dense_buf(var, "red", (var.elements,), torch.float32)
        torch.cuda.synchronize(self.device)

    def prefetch(self, batch: dict) -> None:
        """Build the plans of ``batch`` (the next step's) now, on the current
        stream, so its step skips dedup."""
        if not self.pipelined:
            return
        for name, tab in self.tables.items():
            ids, k = batch[name][0], tab.applied
            self._plan(tab, ids, k % self.plan_slots)
            tab.pending[k] = (ids, k % self.plan_slots, None)

    def predicted_transfer(self) -> TransferReport:
        """The reference's closed-form per-GPU bytes of this plan
        (:func:`transfer.transfer_model`), to print beside the measured ones."""
        from .transfer import transfer_model

        return transfer_model(self.graph, self.plan, self.cluster)

    def _bytes_report(self) -> TransferReport:
        n = self.world_size
        rows = [[0.0, 0.0] for _ in range(n)]
        for name, c in self.last_counts.items():
            eg, ing = wire_bytes(c["send"], c["recv"], self.rank, self.tables[name].D)
            rows[self.rank][0] += eg
            rows[self.rank][1] += ing
        for var in self.dense:
            if n > 1:
                per_dir = 2.0 * var.payload_bytes * (n - 1) / n
                rows[self.rank][0] += per_dir
                rows[self.rank][1] += per_dir
        return TransferReport(tuple(tuple(r) for r in rows))

    def _trace(self) -> tuple:
        out = []
        me = (self.rank, "gpu0")
        for name, c in self.last_counts.items():
            D = self.tables[name].D
            for o in range(self.world_size):
                if c["send"][o]:
                    out.append(Message(me, (o, "server"), c["send"][o] * (8 + 4 * D), name, -1, "push"))
                if c["recv"][o]:
                    out.append(Message((self.rank, "server"), (o, "gpu0"), c["recv"][o] * 4 * D,
                                       name, -1, "pull"))
        return tuple(out)

    def capture(self, batch: dict, warmup: int = 2) -> "ops.StepGraph":
        """Capture one full step on ``batch``'s (static) tensors as a CUDA graph.

        Single-GPU steps have no host synchronisation, so the whole step
        (dedup, apply, gather, dense epilogue) replays with one launch. The
        optimizer struct is baked in at capture: use it for step-independent
        optimizers (SGD / Adagrad); Adam's bias correction would freeze.
        """
        if self.world_size > 1 and self.exchange != "p2p":
            raise NotImplementedError("the NCCL a2a-v path reads counts on the host")
        for tab in self.tables.values():
            tab.pending.clear()
        cur = torch.cuda.current_stream()
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            for _ in range(warmup):
                self.step(batch, timed=False)
        cur.wait_stream(side)
        g = ops.StepGraph(self.graph_node_priority)
        with g.capture():
            self.step(batch, timed=False)
        return g

    def capture_pipelined(self, batches: list, steps_per_graph: int = 1,
                          warm: bool = True) -> list:
        """CUDA graphs over a rotation of batches: graph r applies batches[r]
        with the plan built by the step before and builds the plan of
        batches[r+1]. With ``steps_per_graph`` = G > 1 one graph holds G
        consecutive steps (batches[G·r … G·r+G-1]), so the step boundary inside
        it is a dependency edge instead of a graph launch.

        Replay them in order, repeatedly (and only replay them: the runner's
        host-side plan bookkeeping then describes the replays, not eager
        steps). ``len(batches)`` must be even and a multiple of G; the plan
        lookahead is the deepest L <= ``lookahead`` whose L + 1 slots divide it
        (6 batches: 2 steps ahead). The first plan is built
        eagerly here, followed by one eager rotation that sizes every buffer;
        ``warm=False`` skips both (the caller ran them, e.g. every emulated rank
        of :mod:`.emulate` interleaved, since their waits depend on each other).
        """
        R = len(batches)
        G = steps_per_graph
        if R < 2 or R % 2:
            raise ValueError("capture_pipelined needs an even number (>= 2) of batches")
        if G < 1 or R % G:
            raise ValueError("steps_per_graph must divide the number of batches")
        # slot of step k = k % (L + 1) must be periodic in the rotation: the
        # deepest lookahead L <= self.lookahead with R % (L + 1) == 0
        L = self.lookahead
        while L > 1 and R % (L + 1):
            L -= 1
        if L != self.lookahead:
            if not warm:
                raise ValueError(f"{R} batches do not rotate {self.lookahead + 1} plan slots")
            self.lookahead = L

        def ahead(j):
            return [batches[(j + 1 + i) % R] for i in range(L)]

        if self.world_size > 1 and self.exchange != "p2p":
            raise NotImplementedError("the NCCL a2a-v path reads counts on the host")
        # (the AR-sparse / PS-dense baselines are not pipelined: each graph then
        # plans its own batch; prefetch() and next_batch are no-ops for them)
        if warm:
            for tab in self.tables.values():
                tab.pending.clear()
            self.prefetch(batches[0])
            for r in range(R):  # eager warm-up rotation (sizes every buffer)
                self.step(batches[r], timed=False, upcoming=ahead(r))
            torch.cuda.synchronize()
        graphs = []
        for r in range(0, R, G):
            # plans pending from before this capture: built by the eager warm-up
            # (synchronised) or by the previous graph (which precedes this one in
            # stream order at replay): no event to wait for inside the capture
            for tab in self.tables.values():
                tab.pending = {k: (ids, slot, None) for k, (ids, slot, _) in tab.pending.items()}
            g = ops.StepGraph(self.graph_node_priority)
            self._ps_used = set()
            with g.capture():
                for j in range(r, r + G):
                    self.step(batches[j], timed=False, upcoming=ahead(j))
                self._join_plan_streams()  # a capture ends with every stream joined
            graphs.append(g)
        # the plans left pending were only captured (built at replay time, with
        # captured events): an eager step after this plans inline instead
        for tab in self.tables.values():
            tab.pending.clear()
        return graphs

    # ------------------------------------------------------------------ timing / P search
    def measure_graphs(self, batches: list, iterations: int = 40) -> float:
        """Mean device step time (us) over the second half of ``iterations``
        steps, max over ranks. Steps are pipelined graph replays when possible
        (even ``len(batches)``), eager steps otherwise."""
        R = len(batches)
        graphs = None
        if self.pipelined and R % 2 == 0:
            graphs = self.capture_pipelined(batches)

        def run(k0, k):
            for i in range(k0, k0 + k):
                if graphs:
                    graphs[i % R].replay()
                else:
                    self.step(batches[i % R], timed=False)

        half = max(iterations // 2, 1)
        run(0, half)  # discarded half (warm-up)
        stream = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if self.world_size > 1:
            import torch.distributed as dist

            dist.barrier()
        a.record(stream)
        run(half, iterations - half)
        b.record(stream)
        torch.cuda.synchronize()
        t = a.elapsed_time(b) * 1e3 / max(iterations - half, 1)
        del graphs
        torch.cuda.synchronize()
        if self.world_size > 1:
            import torch.distributed as dist

            x = torch.tensor([t], dtype=torch.float64, device=self.device)
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
            t = float(x.item())
        return t

    def measure(self, make_batch, iterations: int = 100) -> float:
        """Mean device step time (us) with the first half discarded
        (reference `simulate.py:380-402`, `PAPER.md:485`)."""
        if iterations < 2:
            raise SpecError(f"iterations must be >= 2, got {iterations}")
        times = []
        for i in range(iterations):
            stats = self.step(make_batch(i), timed=True)
            times.append(stats.iter_time_us)
        kept = times[iterations // 2:]
        t = float(np.mean(kept))
        if self.world_size > 1:
            import torch.distributed as dist

            x = torch.tensor([t], dtype=torch.float64, device=self.device)
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
            t = float(x.item())
        return t


def simulate_training(plan: DistributedPlan, graph: GraphSpec, cluster: ClusterSpec,
                      profile=None, iterations: int = 100, warmup_inflation: float = 1.5,
                      seed: int = 0, *, rank: int = 0, world_size: int = 1, comm=None,
                      optimizer: OptimizerConfig | None = None, device=None, **kw) -> float:
    """Device counterpart of the reference's ``simulate_training``
    (`sparseplan/simulate.py:380-402`, same signature): the mean time (us) of
    ``iterations`` REAL hybrid steps of ``plan`` on synthetic inputs of the
    graph's shapes (:func:`synth.graph_batches`), the first half discarded
    (`PAPER.md:485`), max over ranks, plus the profile's serialized compute
    time. ``warmup_inflation`` only pins the interface: the discarded warm-up
    half is measured, not modelled. One process per GPU (``comm`` for n > 1)."""
    from .synth import graph_batches

    if iterations < 2:
        raise SpecError(f"iterations must be >= 2, got {iterations}")
    dev = torch.device(device if device is not None else torch.cuda.current_device())
    runner = HybridRunner(plan, graph, cluster, rank=rank, world_size=world_size, comm=comm,
                          optimizer=optimizer, device=dev, seed=seed, **kw)
    try:
        t = runner.measure_graphs(graph_batches(graph, seed, rank, 2, dev), iterations)
    finally:
        runner.close()
    return t + (profile.compute_us_per_gpu if profile is not None else 0.0)


def device_evaluator(graph: GraphSpec, cluster: ClusterSpec, make_batch, *, rank: int = 0,
                     world_size: int = 1, comm=None, optimizer: OptimizerConfig | None = None,
                     iterations: int = 40, names: list | None = None, rotations: int = 2,
                     log: list | None = None, **kw):
    """evaluator(P) -> mean device step time (us), for :func:`tuning.tune_evaluator`.

    Rebuilds the hybrid plan with every partitionable sparse Weight split into P
    (the reference CLI's shared-P rule, `cli.py:93-102`), runs ``iterations``
    real steps (CUDA-graph replays when the exchange allows it) on
    ``rotations`` batches from ``make_batch(i)``, discards the first half
    (`simulate.py:380-402`, `PAPER.md:485`) and returns the mean of the rest,
    max over ranks — so every rank takes the same search decisions.
    """
    cands = names or [v.name for v in graph.variables if v.kind == "sparse" and v.partitionable]

    def evaluator(P: int) -> float:
        parts = {n: min(P, graph.variable(n).elements) for n in cands}
        plan = transform_hybrid(graph, cluster, partitions=parts)
        runner = HybridRunner(plan, graph, cluster, rank=rank, world_size=world_size, comm=comm,
                              optimizer=optimizer, **kw)
        try:
            batches = [make_batch(i) for i in range(rotations)]
            t = runner.measure_graphs(batches, iterations)
        finally:
            runner.close()
            del runner
            torch.cuda.empty_cache()
        if log is not None:
            log.append((P, t))
        return t

    return evaluator
