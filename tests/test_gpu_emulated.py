"""Multi-rank parity on ONE GPU: n emulated ranks (``emulate.LocalWorld``) run
the real peer-memory protocol — worker push epilogue (EpiPush + k_publish),
owner merge (k_owner_scan / k_owner_rows, and the alternative k_owner_apply /
k_owner_stream), k_applied / k_wait, stitch, and the dense K7 over peer memory
(SM stores with uniform and weighted splits, copy engines, the pipelined single
kernel) — with every rank's step in flight on its own stream. Results are
compared BIT-EXACTLY with the oracle: ``coracle.sparse_step`` for tables and
pulled rows (reference PS push/pull + server update, `sparseplan/simulate.py:
183-240,294-323`) and the rank-order fp32 sum for the dense mean (reference
ring allreduce, `simulate.py:97-135`).

This is the coverage the driver's 1-GPU box can see; tests/dist_gpu_check.py
runs the same protocol across real GPUs (one process per GPU, cudaIpc windows).
"""

import json

import numpy as np
import pytest
import torch

from oracle import coracle
from oracle import oracle as orc

pytestmark = pytest.mark.gpu
F32 = np.float32
HPAR = {"lr": 0.2, "beta1": 0.9, "beta2": 0.999, "eps": 1e-8}


def _t(x, dev):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


@pytest.fixture
def knobs(cuda):
    """Set hp_debug_* switches for one test and restore the defaults after."""
    from paper_1808_02621_b200 import _lib

    lib = _lib.load()
    defaults = {"owner_stream": 2, "dar_blocks": 0, "dar_buckets": 1, "dar_rg_blocks": 0, "dar_tma": 36, "dar_rg_tma": 0, "wait_timeout": 0}

    def set_(name, v):
        getattr(lib, f"hp_debug_set_{name}")(v)

    yield set_
    for k, v in defaults.items():
        set_(k, v)


class Emu:
    """n HybridRunners of one process sharing cuda:0, linked by a LocalWorld,
    plus the oracle state of every table."""

    def __init__(self, cuda, n, tables, dense, opt, dense_exchange, P=8, dense_dtype=torch.float32,
                 seed=3, concurrent=False, dense_in_dtype=torch.float32):
        import paper_1808_02621_b200 as hp
        from paper_1808_02621_b200.emulate import LocalWorld
        from paper_1808_02621_b200.synth import Workload

        self.dev, self.n, self.opt = cuda, n, opt
        self.wl = Workload("emu", tables, dense, {"kind": opt, "lr": HPAR["lr"], "init_acc": 0.1},
                           2560, partitions=P)
        self.graph = hp.load_graph_spec(json.dumps(self.wl.graph_json()))
        cluster = hp.ClusterSpec.b200_box(n)
        self.plan = hp.transform_hybrid(self.graph, cluster, partitions={t.name: P for t in tables})
        world = LocalWorld(n)
        optc = hp.OptimizerConfig(kind=opt, lr=HPAR["lr"], init_acc=0.1)
        self.runners = [hp.HybridRunner(self.plan, self.graph, cluster, rank=r, world_size=n,
                                        comm=world.comm(r), optimizer=optc, device=cuda, seed=seed,
                                        dense_exchange=dense_exchange, dense_dtype=dense_dtype,
                                        dense_in_dtype=dense_in_dtype)
                        for r in range(n)]
        self.dense_in_dtype = dense_in_dtype
        if not concurrent:  # one stream per rank (emulate.LocalWorld.serialize)
            for run in self.runners:
                LocalWorld.serialize(run)
        self.streams = [torch.cuda.Stream(device=cuda) for _ in range(n)]  # created back to back
        self.seed = seed
        self.dense_dtype = dense_dtype
        self.states = None
        self.step_no = 0

    def batches(self, seed, empty=()):
        from paper_1808_02621_b200.synth import make_batch

        host = []
        for r in range(self.n):
            b = make_batch(self.wl, seed=seed, rank=r)
            if r in empty:
                for t in self.wl.tables:
                    b[t.name] = (np.zeros(0, np.int64), np.zeros((0, t.D), F32))
            host.append(b)
        dev = [{k: ((_t(v[0], self.dev), _t(v[1], self.dev)) if isinstance(v, tuple)
                    else _t(v, self.dev)) for k, v in b.items()} for b in host]
        if self.dense_in_dtype == torch.bfloat16:  # bf16 gradients; the oracle sees their fp32 value
            for b, d in zip(host, dev):
                for name in self.wl.dense:
                    g16 = torch.from_numpy(b[name]).to(torch.bfloat16)
                    b[name] = g16.float().numpy()
                    d[name] = g16.to(self.dev)
        return host, dev

    def init_oracle(self, host_batches_all):
        """Lazy oracle tables, initialised at every row any of the batches touches."""
        names = [v.name for v in self.graph.variables]
        self.states = {}
        for t in self.wl.tables:
            touched = np.concatenate([b[t.name][0] for b in host_batches_all])
            i = names.index(t.name)
            self.states[t.name] = orc.lazy_state(self.opt, t.V, t.D, self.seed * 1000 + i, touched)
        self.touched = {t.name: np.unique(np.concatenate([b[t.name][0] for b in host_batches_all]))
                        for t in self.wl.tables}

    def oracle_step(self, host):
        """Advance the oracle one step; returns the expected pulled rows / dense out."""
        self.step_no += 1
        outs = {}
        for t in self.wl.tables:
            owner = self.plan.owner_table(t.name)
            res = coracle.sparse_step(self.states[t.name], self.opt, HPAR, self.step_no,
                                      [b[t.name] for b in host], t.V, self.wl.partitions, owner)
            outs[t.name] = [res[r]["out"] for r in range(self.n)]
        for name in self.wl.dense:
            d = coracle.dense_mean([b[name] for b in host], F32(1.0 / self.n))
            outs[name] = torch.from_numpy(d).to(self.dense_dtype)
        return outs

    def check_outputs(self, ref):
        for t in self.wl.tables:
            for r, run in enumerate(self.runners):
                got = run.outputs[t.name].cpu().numpy()
                assert np.array_equal(got, ref[t.name][r]), (t.name, r)
        for name in self.wl.dense:
            for r, run in enumerate(self.runners):
                got = run.dense_out[name].reshape(-1)
                assert torch.equal(got.cpu(), ref[name]), (name, r)

    def table_rows(self, name, rows, k=None):
        """Rows ``rows`` of table ``name`` (w, or optimizer state k) gathered from
        their owners' slabs."""
        tab0 = self.runners[0].tables[name]
        b = tab0.bounds
        p = np.searchsorted(b, rows, side="right") - 1
        own = tab0.owner[p]
        out = np.empty((len(rows), tab0.D), F32)
        for r, run in enumerate(self.runners):
            sel = own == r
            if not sel.any():
                continue
            tab = run.tables[name]
            srow = tab.part_base_host[p[sel]] + rows[sel] - b[p[sel]]
            src = tab.w if k is None else tab.state[k]
            out[sel] = src[_t(srow, self.dev)].cpu().numpy()
        return out

    def check_tables(self):
        for t in self.wl.tables:
            rows = self.touched[t.name]
            rows = rows[(rows >= 0) & (rows < t.V)]
            st = self.states[t.name]
            assert np.array_equal(self.table_rows(t.name, rows), st["w"][rows]), t.name
            if self.opt == "adagrad":
                assert np.array_equal(self.table_rows(t.name, rows, 0), st["acc"][rows])
            if self.opt == "adam":
                assert np.array_equal(self.table_rows(t.name, rows, 0), st["m"][rows])
                assert np.array_equal(self.table_rows(t.name, rows, 1), st["v"][rows])

    def errors(self):
        for run in self.runners:
            run.check_errors(sync=True)

    def close(self):
        torch.cuda.synchronize()
        for run in self.runners:
            run.close()


def _small_tables():
    from paper_1808_02621_b200.synth import TableShape

    return [TableShape("embedding", 60_000, 128, 2560),
            TableShape("softmax", 60_000, 256, 2560, sampled=2048)]


def _eager_pipelined(emu, seeds, empty=()):
    """Eager steps: first without a prefetched plan, then pipelined (the plan of
    step i+1 built on the plan stream during step i)."""
    from paper_1808_02621_b200.emulate import step_all

    data = [emu.batches(s, empty) for s in seeds]
    emu.init_oracle([b for h, _ in data for b in h])
    step_all(emu.runners, emu.streams, data[0][1])
    emu.check_outputs(emu.oracle_step(data[0][0]))
    for run, b in zip(emu.runners, data[1][1]):
        run.prefetch(b)
    for i in range(1, len(data)):
        nxt = data[i + 1][1] if i + 1 < len(data) else None
        step_all(emu.runners, emu.streams, data[i][1], nxt)
        emu.check_outputs(emu.oracle_step(data[i][0]))
    emu.check_tables()
    emu.errors()


@pytest.mark.parametrize("n,ctas,rg", [(2, 3, 0), (4, 1, 0), (3, 0, 0), (2, 32, 5), (3, 32, 2)])
def test_emulated_dense_tma_scatter_bit_exact(cuda, knobs, n, ctas, rg):
    """The SM-store dense exchange with its scatter on TMA bulk copies (few
    CTAs), by LSU stores (0), and with the reduce/gather on TMA (rg CTAs)."""
    knobs("dar_tma", ctas)
    knobs("dar_rg_tma", rg)
    emu = Emu(cuda, n, _small_tables(), {"lstm": 100_000}, "adagrad", "p2p-sm")
    try:
        _eager_pipelined(emu, [1, 2, 3])
    finally:
        emu.close()


@pytest.mark.parametrize("n,out_dtype", [(2, torch.float32), (3, torch.bfloat16)])
def test_emulated_bf16_dense_gradients_bit_exact(cuda, n, out_dtype):
    """bf16 dense gradients (in_dtype) over the SM-store exchange: bf16 on the
    links, widened exactly, summed in rank order in fp32, scaled, cast."""
    emu = Emu(cuda, n, _small_tables(), {"lstm": 100_000}, "adagrad", "p2p-sm",
              dense_dtype=out_dtype, dense_in_dtype=torch.bfloat16)
    try:
        _eager_pipelined(emu, [1, 2, 3])
    finally:
        emu.close()


@pytest.mark.parametrize("n,buckets,opt", [(2, 2, "adagrad"), (3, 5, "sgd"), (4, 3, "adam")])
def test_emulated_dense_buckets_bit_exact(cuda, knobs, n, buckets, opt):
    """The SM-store dense exchange with its phases cut into `buckets` pieces per
    chunk (per-bucket epochs): same rank-order sums as one bucket."""
    knobs("dar_buckets", buckets)
    emu = Emu(cuda, n, _small_tables(), {"lstm": 100_000}, opt, "p2p-sm")
    try:
        _eager_pipelined(emu, [1, 2, 3])
    finally:
        emu.close()


@pytest.mark.parametrize("n,dense_exchange,opt,concurrent",
                         [(2, "p2p-sm", "adagrad", True),    # the multi-stream step
                          (2, "p2p-sm", "adagrad", False),
                          (4, "p2p-sm", "adagrad", False),   # weighted split
                          (8, "p2p-sm", "adagrad", False),   # a full box (the driver's N=8 run)
                          (3, "p2p", "sgd", False),          # copy engines
                          (2, "p2p-pipe", "adam", True),
                          (2, "p2p-pull", "adagrad", True),  # one-shot pull (n = 2 default)
                          (3, "p2p-pull", "sgd", False),
                          (4, "p2p-pipe", "adagrad", False)])
def test_emulated_hybrid_steps_bit_exact(cuda, knobs, n, dense_exchange, opt, concurrent):
    if dense_exchange == "p2p-pipe":
        knobs("dar_blocks", 24)  # n persistent kernels share one GPU: keep them co-resident
    emu = Emu(cuda, n, _small_tables(), {"lstm": 100_000}, opt, dense_exchange,
              concurrent=concurrent)
    try:
        if n >= 4 and dense_exchange == "p2p-sm":
            assert emu.runners[0].dense_weights is not None  # hot-owner split in use
        _eager_pipelined(emu, [1, 2, 3])
    finally:
        emu.close()


def test_emulated_forward_pull_reads_owner_slabs(cuda):
    """HybridRunner.pull at n > 1 (hp_xchg_pull): after hybrid steps every rank
    reads the current rows of any ids — homed anywhere — straight from the
    owners' slabs (peer loads); dropped ids give zero rows."""
    emu = Emu(cuda, 4, _small_tables(), {"lstm": 40_000}, "adagrad", "p2p-sm")
    try:
        _eager_pipelined(emu, [21, 22])
        rng = np.random.default_rng(5)
        for t in emu.wl.tables:
            pool = emu.touched[t.name]
            ids = rng.choice(pool, 3000)
            ids[:7] = [-1, t.V, t.V + 5, -9, 0, 1, 2]
            ref = orc.pull_rows(emu.states[t.name]["w"], ids)
            ref[4:7] = emu.table_rows(t.name, np.array([0, 1, 2]))  # untouched rows: device init
            for r, run in enumerate(emu.runners):
                got = run.pull(t.name, _t(ids, emu.dev)).cpu().numpy()
                ok = np.isin(ids, pool) | (ids < 0) | (ids >= t.V) | (ids <= 2)
                assert np.array_equal(got[ok], ref[ok]), (t.name, r)
    finally:
        emu.close()


@pytest.mark.parametrize("owner_kernel", [0, 1])
def test_emulated_alternative_owner_kernels(cuda, knobs, owner_kernel):
    """k_owner_apply (0) and k_owner_stream (1) instead of the two-pass default."""
    knobs("owner_stream", owner_kernel)
    emu = Emu(cuda, 2, _small_tables(), {"lstm": 40_000}, "adagrad", "p2p-sm")
    try:
        _eager_pipelined(emu, [4, 5])
    finally:
        emu.close()


def test_emulated_empty_rank_and_bf16_dense(cuda):
    """A rank with empty IndexedSlices still publishes and waits every step (its
    next push must follow every owner's apply); dense output cast to bf16."""
    emu = Emu(cuda, 4, _small_tables(), {"lstm": 100_000}, "adagrad", "p2p-sm",
              dense_dtype=torch.bfloat16)
    try:
        _eager_pipelined(emu, [6, 7, 8], empty=(2,))
    finally:
        emu.close()


@pytest.mark.parametrize("n,R", [(2, 2), (4, 2), (2, 6)])
def test_emulated_graph_replays_bit_exact(cuda, n, R):
    """The pipelined CUDA-graph rotation (bench.py's timed path) of every rank,
    replayed concurrently, with 1 and 2 steps per graph; R = 6 batches run
    the plans 2 steps ahead (3 plan slots), R = 2 one step ahead."""
    from paper_1808_02621_b200.emulate import capture_pipelined_all, replay_all

    emu = Emu(cuda, n, _small_tables(), {"lstm": 100_000}, "adagrad", "p2p-sm",
              concurrent=n == 2)
    try:
        data = [emu.batches(s) for s in range(11, 11 + R)]
        emu.init_oracle([b for h, _ in data for b in h])
        rot = [[data[k][1][r] for k in range(R)] for r in range(n)]
        graphs = capture_pipelined_all(emu.runners, emu.streams, rot)  # eager rotation
        assert emu.runners[0].lookahead == (2 if R == 6 else 1)
        for k in range(R):
            emu.oracle_step(data[k][0])
        for _ in range(2):
            for k in range(R):
                replay_all(graphs, emu.streams, k)
                emu.check_outputs(emu.oracle_step(data[k][0]))
        multi = capture_pipelined_all(emu.runners, emu.streams, rot, steps_per_graph=2)
        for k in range(R):
            emu.oracle_step(data[k][0])
        for g in range(R // 2):
            replay_all(multi, emu.streams, g)
            emu.oracle_step(data[2 * g][0])
            emu.check_outputs(emu.oracle_step(data[2 * g + 1][0]))
        emu.check_tables()
        emu.errors()
        del graphs, multi
    finally:
        emu.close()


def test_emulated_lm1b_exact_shapes_n2(cuda):
    """BASELINE configs[1] shapes across 2 emulated ranks: two 800k x 512 fp32
    tables, T = 2560 (embedding) and 2560 + 8192 sampled (softmax) per worker,
    9.4M dense, Adagrad, P = 8; every pulled row, touched table/accumulator row
    and the dense mean bit-exact."""
    from paper_1808_02621_b200.synth import WORKLOADS

    lm = WORKLOADS["lm1b"]
    emu = Emu(cuda, 2, lm.tables, dict(lm.dense), "adagrad", "p2p-sm", concurrent=True)
    try:
        _eager_pipelined(emu, [1, 2])
    finally:
        emu.close()


def test_emulated_push_timeout_raises(cuda, knobs):
    """A rank whose peer never pushes: its waits time out (bounded, no hang),
    the owner merges NOTHING from the partial inboxes, and step() raises."""
    from paper_1808_02621_b200._lib import HybridPathError

    knobs("wait_timeout", 20_000_000)  # ~10 ms
    emu = Emu(cuda, 2, _small_tables()[:1], {"lstm": 4096}, "sgd", "p2p-sm")
    try:
        _, dev = emu.batches(1)
        w0 = emu.runners[0].tables["embedding"].w.clone()
        with torch.cuda.stream(emu.streams[0]):
            emu.runners[0].step(dev[0], timed=False)  # rank 1 never steps
        torch.cuda.synchronize()
        assert torch.equal(emu.runners[0].tables["embedding"].w, w0)  # nothing applied
        with pytest.raises(HybridPathError, match="push wait timed out"):
            emu.runners[0].check_errors(sync=True)
    finally:
        emu.close()
