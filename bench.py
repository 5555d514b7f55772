#!/usr/bin/env python
"""Hybrid-step benchmark (BASELINE.json metric) — one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload lm1b] [--impl ours|reference]

N=1 runs in-process; N>1 is launched by the driver with torch.distributed.run
(one rank per GPU, NCCL). A "step" is one hybrid-communication pass over one
batch per worker: dense allreduce(+scale/cast) and, per sparse table, dedup ->
route -> (exchange) -> merge + Adagrad apply -> gather/pull -> stitch.

value : words/s = N * 2560 * K / t, t = max over ranks of the device time of
        K steps with inputs resident in HBM (rotated over R pre-generated
        batches whose total exceeds L2, so no step reads warm inputs).
e2e   : the same metric through HybridRunner with the step's inputs copied
        from pinned host memory inside the timed region and a result read back.
roofline : the K4 scatter-apply kernel of the largest table, algorithmic bytes
         / its CUDA-event duration, against MEASURED_PEAKS.json.
cpu_baseline : the oracle port (oracle/hp_oracle.c, OpenMP, all host threads) timed on
               this host (rank 0, N=1).
--impl reference : the oracle port on this host for the same config/metric.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "hybrid-step words/sec"
UNIT = "words/s"


def metric_for(wl, world: int):
    """(metric, unit, units per step of the whole job, per-batch helper).

    LM/NMT-shaped workloads: words/s (n * 2560 per step). Sparse
    microbench: unique sparse rows/s summed over workers. Dense-only: allreduce
    bus GB/s = 2(n-1)/n * S * 4 / t (NCCL-tests convention; HBM GB/s at n=1).
    """
    if wl.words_per_worker:
        return METRIC, UNIT
    if wl.tables:
        return "sparse rows/sec", "rows/s"
    return "dense allreduce bus GB/s", "GB/s"


def units_per_step(wl, world: int, host_batches, rank: int) -> float:
    if wl.words_per_worker:
        return float(world * wl.words_per_worker)
    if wl.tables:
        u = np.mean([sum(len(np.unique(b[t.name][0])) for t in wl.tables) for b in host_batches])
        return float(u) * world  # approximation until all-reduced below
    S = sum(wl.dense.values()) * 4
    return (2.0 * (world - 1) / world * S if world > 1 else 2.0 * S) / 1e9


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="lm1b")
    ap.add_argument("--partitions", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rotations", type=int, default=0, help="distinct resident batches")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--steps-per-graph", type=int, default=6,
                    help="consecutive steps captured in one CUDA graph (divides the rotation); "
                         "graphs of 3 and 2 steps cover the remainder")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"])
    ap.add_argument("--dense-exchange", default=None,
                    choices=["p2p", "p2p-sm", "p2p-pipe", "p2p-pull", "nvls", "nccl"])
    ap.add_argument("--dense-in", default="f32", choices=["f32", "bf16"],
                    help="dtype the dense gradients arrive in (not BASELINE's config: an "
                         "in_dtype data point; bf16 travels as bf16 over the SM-store exchange)")
    ap.add_argument("--dense-split", default="auto",
                    help="peer-memory dense exchange: reduction share per rank "
                         "('auto', 'uniform' or comma-separated weights)")
    ap.add_argument("--arch", default="hybrid", choices=["hybrid", "ar", "ps"],
                    help="mechanism plan: transform_hybrid (default) / transform_ar / transform_ps")
    ap.add_argument("--check", action="store_true",
                    help="N=1: before timing, run the bench's own pipelined-graph path on its "
                         "workload against the C oracle (oracle/check.py), bit-exact")
    ap.add_argument("--knob", action="append", default=[],
                    help="instrumentation A/B: NAME=INT calls hp_debug_set_NAME(INT)")
    return ap.parse_args()


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "src": "fallback (B200_PROFILING.md)"}


def k4_traffic(workload: str, table: str):
    """DRAM bytes (read + write) per K4 launch pair from the committed ncu capture
    (profiles/r1b_k4_traffic.json), for the workload/table it was taken on."""
    p = next((q for q in (ROOT / "profiles" / "r2_k4_traffic.json",
                          ROOT / "profiles" / "r1b_k4_traffic.json") if q.exists()), None)
    if p is None:
        return None
    d = json.loads(p.read_text())
    if d.get("workload") != workload or d.get("table") != table:
        return None
    return d["traffic_bytes_per_launch"]


# ------------------------------------------------------------------ clocks
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            self.p.wait()

    def summary(self) -> dict:
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = [r.split(",") for r in Path(self.f.name).read_text().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) > 8 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 8 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) > 8 for i in range(4)
                          if r[5 + i].strip().lower() == "active"})
        load = [s for s in sm if mx and s >= 0.3 * max(mx)] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ------------------------------------------------------------------ CPU oracle step
def cpu_oracle_step(wl, batches, states, step):
    """The oracle's hybrid step for len(batches) simulated workers (one process),
    on the OpenMP C restatement (oracle/hp_oracle.c, bit-identical to the numpy
    oracle; tests/test_oracle.py)."""
    from oracle import coracle, oracle as orc

    n = len(batches)
    for t in wl.tables:
        owner = np.zeros(1, np.int32) if n == 1 else orc.owner_table(t.name, wl.partitions, n)
        P = 1 if n == 1 else wl.partitions
        coracle.sparse_step(states[t.name], wl.optimizer["kind"], wl.optimizer, step,
                            [b[t.name] for b in batches], t.V, P, owner)
    for name in wl.dense:
        coracle.dense_mean([b[name] for b in batches], 1.0 / n)


def cpu_threads() -> int:
    from oracle import coracle

    return coracle.threads()


def lazy_states(wl):
    st = {}
    for t in wl.tables:
        z = lambda: np.zeros((t.V, t.D), np.float32)  # calloc: only touched pages are real
        kind = wl.optimizer["kind"]
        st[t.name] = {"w": z()} | ({"acc": z()} if kind == "adagrad" else {}) | (
            {"m": z(), "v": z()} if kind == "adam" else {})
    return st


def time_cpu(wl, n_workers: int, steps: int, seed: int = 0):
    from paper_1808_02621_b200.synth import make_batch

    batches = [make_batch(wl, seed, r) for r in range(n_workers)]
    states = lazy_states(wl)
    cpu_oracle_step(wl, batches, states, 1)  # warm-up (page faults, caches)
    t0 = time.perf_counter()
    for s in range(steps):
        cpu_oracle_step(wl, batches, states, s + 2)
    dt = (time.perf_counter() - t0) / steps
    words = n_workers * wl.words_per_worker
    return words / dt, dt


def run_reference(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.gpus
    _, dt = time_cpu(wl, n, max(args.steps, 1), seed=0)
    from paper_1808_02621_b200.synth import make_batch

    metric, unit = metric_for(wl, n)
    value = units_per_step(wl, n, [make_batch(wl, 0, 0)], 0) / dt
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": config(args, wl),
        "cpu_baseline": {"value": value, "unit": unit, "cores": cpu_threads(), "kind": "port",
                         "sample": f"{args.steps} full oracle steps of {n} simulated worker(s), "
                                   f"C restatement, OpenMP x{cpu_threads()}"},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config(args, wl):
    return {"workload": wl.name, "tables": [f"{t.name}:{t.V}x{t.D},T={t.T + t.sampled}"
                                            for t in wl.tables],
            "dense_elems": sum(wl.dense.values()), "optimizer": wl.optimizer["kind"],
            "partitions": args.partitions or wl.partitions, "words_per_worker": wl.words_per_worker,
            "parallelism": f"{args.arch} dp{args.gpus}",
            "l2_policy": "inputs rotated over distinct resident batches totalling > 2x L2"}


# ------------------------------------------------------------------ GPU arm
_T0 = time.time()


def _mark(msg: str) -> None:
    """Wall-clock progress on stderr (where a multi-minute run spends its time)."""
    print(f"[bench {time.time() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def main():
    args = parse()
    from paper_1808_02621_b200.synth import WORKLOADS, micro_workload

    wl = WORKLOADS[args.workload] if not args.workload.startswith("micro") else micro_workload(
        int(args.workload.split("_")[1]))
    if args.impl == "reference":
        return run_reference(args, wl)
    knobs = args.knob + [kv for kv in os.environ.get("HP_KNOBS", "").split(",") if kv]
    if knobs:
        from paper_1808_02621_b200 import _lib

        for kv in knobs:
            k, v = kv.split("=")
            getattr(_lib.load(), f"hp_debug_set_{k}")(int(v))

    import torch
    import torch.distributed as dist

    import paper_1808_02621_b200 as hp
    from paper_1808_02621_b200 import ops
    from paper_1808_02621_b200.synth import make_batch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = hp.Comm.from_torch_distributed()
    P = args.partitions or wl.partitions
    graph = hp.load_graph_spec(json.dumps(wl.graph_json()))
    cluster = hp.ClusterSpec.b200_box(world)
    parts = {t.name: P for t in wl.tables}
    if args.arch == "ar":  # SURVEY §8f baselines: the same Weights under AR / PS
        plan = hp.transform_ar(graph, cluster)
    elif args.arch == "ps":
        plan = hp.transform_ps(graph, cluster, local_agg=True, partitions=parts)
    else:
        plan = hp.transform_hybrid(graph, cluster, partitions=parts)
    opt = hp.OptimizerConfig(**wl.optimizer)
    runner = hp.HybridRunner(plan, graph, cluster, rank=rank, world_size=world, comm=comm,
                             optimizer=opt, device=dev, seed=0, exchange=args.exchange,
                             dense_exchange=args.dense_exchange,
                             dense_split=(args.dense_split if args.dense_split in ("auto", "uniform")
                                          else [float(x) for x in args.dense_split.split(",")]),
                             dense_in_dtype=torch.bfloat16 if args.dense_in == "bf16" else torch.float32)
    if args.dense_in == "bf16" and args.check:
        raise SystemExit("--check runs the BASELINE config (fp32 dense gradients)")

    # resident batches, rotated so their total exceeds 2x L2 (126 MB)
    host = [make_batch(wl, seed=1 + i, rank=rank) for i in range(1)]
    per_batch = sum(v[0].nbytes + v[1].nbytes if isinstance(v, tuple) else v.nbytes
                    for v in host[0].values())
    R = args.rotations or max(2, int(np.ceil(2 * 126e6 / max(per_batch, 1))))
    # the pipelined graphs rotate lookahead + 1 plan slots (plans built 2 steps
    # ahead: 3 slots) and the rotation must be even: a multiple of 6
    R = min(-(-R // 6) * 6, 18) if not args.rotations else R
    host += [make_batch(wl, seed=1 + i, rank=rank) for i in range(1, R)]

    din = runner.dense_in_dtype

    def to_dev(b):
        return {k: ((torch.from_numpy(v[0]).to(dev), torch.from_numpy(v[1]).to(dev))
                    if isinstance(v, tuple) else torch.from_numpy(v).to(din).to(dev))
                for k, v in b.items()}

    batches = [to_dev(b) for b in host]
    _mark("inputs resident")
    use_graph = (world == 1 or args.exchange == "p2p") and not args.no_graph
    stream = torch.cuda.current_stream()
    check = None
    if args.check and world == 1:  # parity of this exact config, before (not in) the timing
        from oracle.check import check_runner_n1

        G0 = args.steps_per_graph if R % max(args.steps_per_graph, 1) == 0 else 1
        check = check_runner_n1(runner, wl, host, batches, steps_per_graph=G0, replays=1)
        check = {"ok": True, "vs": "C oracle (oracle/check.py), bit-exact"} | check

    for i in range(args.warmup):
        runner.step(batches[i % R], timed=False)
    torch.cuda.synchronize()
    l0 = ops.launch_count()
    runner.step(batches[0], timed=False)
    torch.cuda.synchronize()
    launches_per_step = ops.launch_count() - l0
    # Graph r applies batch r with the plan graph r-1 built, and builds batch r+1's
    # plan on a side stream meanwhile (plans depend only on the ids).
    graphs = runner.capture_pipelined(batches) if use_graph else None
    _mark("graphs captured")
    G = args.steps_per_graph if graphs and R % max(args.steps_per_graph, 1) == 0 else 1
    # G > 1: graphs of G consecutive steps (same rotation and plan-slot order as
    # the single-step graphs), so K steps replay as K // G launches; the
    # remainder replays graphs of 3 / 2 steps where they divide the rotation,
    # then single steps. (Measured LM1B N=1 per step: 1 step per graph 51.3 us,
    # 2: 41, 3: 38.2, 6: 36.2 - each graph ends by joining the plan streams.)
    multis = {}
    rem = os.environ.get("HP_BENCH_REMAINDER", "1") == "1"
    for g in sorted({G, 3, 2} if rem else {G}, reverse=True):
        if G > 1 and 1 < g <= G and R % g == 0:
            multis[g] = runner.capture_pipelined(batches, steps_per_graph=g)
    torch.cuda.synchronize()
    pos = [0]  # next step's index in the rotation

    def run_steps(k):
        done = 0
        while done < k:
            i = pos[0]
            g = next((g for g in multis if i % g == 0 and k - done >= g), 0)
            if g:
                multis[g][(i % R) // g].replay()
                n = g
            elif graphs:
                graphs[i % R].replay()
                n = 1
            else:
                runner.step(batches[i % R], timed=False)
                n = 1
            pos[0] = (i + n) % R
            done += n

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # setup (untimed, before the warm-up): every captured graph replayed once
    # (a graph's first launch uploads it: ~0.1-0.2 ms that must not land in the
    # timed region), each set over a whole rotation so the position stays 0;
    # then align the rotation so the warm-up ends on a G-step graph boundary
    for gs in list(multis.values()) + ([graphs] if graphs else []):
        for gr in gs:
            gr.replay()
    run_steps((-max(args.warmup, 3)) % G)
    run_steps(max(args.warmup, 3))
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run_steps(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
    t_dev = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    _mark("timed region done")
    metric, unit = metric_for(wl, world)
    ups = units_per_step(wl, world, host, rank)
    if wl.tables and not wl.words_per_worker and world > 1:  # exact sum of unique rows
        t_u = torch.tensor([ups / world], dtype=torch.float64, device=dev)
        dist.all_reduce(t_u)
        ups = float(t_u.item())
    value = ups * args.steps / t_dev

    # ---- per-kernel timing (eager steps, events around each phase's launches)
    kern = {}
    if world == 1 or runner.exchange == "p2p":
        # Eager steps, tables one after another, each step queued behind a GPU
        # sleep so the CPU enqueue cost never shows up between an event pair;
        # with several ranks every step starts after a barrier (same sleep on
        # every GPU) and each phase reports the max over ranks.
        runner.kernel_events = {}
        runner.concurrent_tables = False
        kt = min(args.steps, 20)
        for i in range(kt):
            if world > 1:
                barrier()
                torch.cuda.synchronize()
            torch.cuda._sleep(20_000_000)
            runner.step(batches[i % R], timed=False)
        torch.cuda.synchronize()
        runner.concurrent_tables = True
        for key, evs in sorted(runner.kernel_events.items()):
            d = [a.elapsed_time(b) * 1e3 for a, b in zip(evs[0::2], evs[1::2])]
            kern[key] = max_over_ranks(float(np.mean(d)))
        runner.kernel_events = None

    # ---- N > 1: the sparse exchange's NVLink bytes (measured from the device
    # send / receive counts of one timed step) against the push / apply kernel
    # times above, and the reference's predicted per-GPU bytes beside them
    sparse_x = None
    if world > 1 and wl.tables and runner.exchange == "p2p":
        st_ = runner.step(batches[0], timed=True)
        mine = torch.tensor(list(st_.per_machine_bytes.per_machine[rank]), dtype=torch.float64,
                            device=dev)
        allb = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allb, mine)
        measured = [[float(x) for x in t.tolist()] for t in allb]
        pred = runner.predicted_transfer().per_machine
        push_b, ret_b = 0.0, 0.0
        for name, c in runner.last_counts.items():
            D = runner.tables[name].D
            push_b += sum(c["send"][o] * (8 + 4 * D) for o in range(world) if o != rank)
            ret_b += sum(c["recv"][s_] * 4 * D for s_ in range(world) if s_ != rank)
        push_max = max_over_ranks(push_b)
        ret_max = max_over_ranks(ret_b)
        t_push = sum(v for k_, v in kern.items() if k_.startswith("push:"))
        t_apply = sum(v for k_, v in kern.items() if k_.startswith("apply:"))
        sparse_x = {
            "push_bytes_max_rank": push_max, "push_us": t_push,
            "push_egress_gbs": push_max / (t_push * 1e-6) / 1e9 if t_push else None,
            "return_bytes_max_rank": ret_max, "apply_return_us": t_apply,
            "return_egress_gbs": ret_max / (t_apply * 1e-6) / 1e9 if t_apply else None,
            "nvlink_peak_gbs": 770.0,
            "note": "push = reduce + NVLink stores (k_reduce EpiPush + k_publish); return = owner "
                    "merge + apply + stores back (k_owner_scan/rows + k_applied): each kernel also "
                    "reads HBM, so egress/t is a lower bound of the link rate",
            "measured_bytes_per_gpu": measured,
            "predicted_bytes_per_gpu_transfer_model": [list(r) for r in pred],
            "predicted_note": "reference transfer_model (uniform alpha, rows only, dense 2(n-1)/n S); "
                              "measured counts ids + rows of the actual Zipf batch: reported, not asserted"}
    pk = peaks()
    roof = None
    big = max(wl.tables, key=lambda t: (t.T + t.sampled) * t.D) if wl.tables else None
    if big is not None and f"k4:{big.name}" in kern:
        tab = runner.tables[big.name]
        T = big.T + big.sampled
        ops.apply_plan_build(batches[0][big.name][0], tab.slab(), tab.ws)
        U = int(tab.ws.buf[:4].view(torch.int32).item())
        k = 1 + opt.n_state
        # K4 + K5 (world 1: apply with the pull fused, hp_apply_plan_pull): gradient
        # rows + positions read, each unique row's state read + written (k tensors),
        # every position's pulled row written. Other worlds: K4 alone.
        fused_pull = world == 1
        algo = T * (4 + 4 * big.D) + U * (4 + 4 * big.D * 2 * k)
        if fused_pull:
            algo += T * 4 * big.D
        us = kern[f"k4:{big.name}"]
        achieved = algo / (us * 1e-6) / 1e9
        roof = {"kernel": (f"K4+K5 merge+apply+pull ({big.name}: split apply - k_reduce short items "
                           "with the pull on a side stream; long chunks -> k_combine -> k_bcast_rows)"
                           if fused_pull else
                           f"K4 merge+apply ({big.name})"), "bound": "hbm",
                "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": k4_traffic(wl.name, big.name),
                "algorithmic_bytes": algo, "launch_us": us, "peak_src": pk["src"],
                "unique_rows": U, "T": T,
                "step_share": us / (t_dev / args.steps * 1e6)}
        gk = f"k5:{big.name}"
        if gk in kern:  # the pull through the plan: positions + unique rows read + rows written
            g_algo = T * 4 + U * 4 * big.D + T * 4 * big.D
            roof["gather"] = {"launch_us": kern[gk], "algorithmic_bytes": g_algo,
                              "achieved": g_algo / (kern[gk] * 1e-6) / 1e9}
        # the whole step against HBM: every kernel's algorithmic bytes once
        # (K4 + K5 per table, + the dense scale/cast in + out only when it runs:
        # at n = 1 with fp32 'mean' K7 is a no-op and launches nothing; dedup < 1%)
        step_bytes = 0.0 if runner.dense_is_noop() else 2.0 * sum(wl.dense.values()) * 4
        for t in wl.tables:
            tb = runner.tables[t.name]
            Tt = t.T + t.sampled
            ops.apply_plan_build(batches[0][t.name][0], tb.slab(), tb.ws)
            Ut = int(tb.ws.buf[:4].view(torch.int32).item())
            step_bytes += Tt * (4 + 4 * t.D) + Ut * (4 + 4 * t.D * 2 * k) + Tt * 4 * t.D
        step_us = t_dev / args.steps * 1e6
        roof["step"] = {"algorithmic_bytes": step_bytes, "us": step_us,
                        "achieved": step_bytes / (step_us * 1e-6) / 1e9,
                        "frac": step_bytes / (step_us * 1e-6) / 1e9 / pk["hbm_gbs"]}

    # ---- N > 1: NVLink roofline of K7 (the dense exchange, the step's critical
    # path), timed alone with events: every rank starts together (barrier + a
    # queued sleep), max over ranks, median of 10. Bytes = the most any rank
    # must send over NVLink for the transport and split in use.
    if world > 1 and wl.dense and not runner.dense_ps:
        S = sum(v.elements for v in runner.dense) * 4
        w = runner.dense_weights or [1.0] * world
        if runner.dense_exchange == "p2p-pull":
            egress = (world - 1) * S
            how = "each rank reads every peer's copy: (n-1) S per rank (ingress)"
        elif runner.dense_exchange in ("p2p", "p2p-sm", "p2p-pipe"):
            c = [x / sum(w) * S for x in w]
            ib = 0.5 if runner.dense_in_dtype == torch.bfloat16 else 1.0  # bf16 scatter: half
            ob = runner.dense_dtype.itemsize / 4
            egress = max((S - c[r]) * ib + (world - 1) * c[r] * ob for r in range(world))
            how = ("max over ranks of (S - chunk_r) * in_bytes/4 + (n-1) chunk_r * out_bytes/4 "
                   "(S, chunks in fp32 bytes)")
        else:
            egress = 2.0 * (world - 1) / world * S
            how = "ring-equivalent bus bytes 2(n-1)/n S"
        def time_k7(replay):
            ts = []
            for i in range(10):
                barrier()
                torch.cuda._sleep(2_000_000)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                replay(i)
                b.record(stream)
                torch.cuda.synchronize()
                ts.append(max_over_ranks(a.elapsed_time(b) * 1e3))
            return float(np.median(ts))

        us_eager = time_k7(lambda i: runner._dense(batches[i % R]))
        # the exchange as the step runs it: captured in a CUDA graph (its 4-6
        # kernels without eager launch gaps), replayed on every rank together
        us_graph = None
        try:
            kg = torch.cuda.CUDAGraph()
            side_ = torch.cuda.Stream(device=dev)
            side_.wait_stream(stream)
            with torch.cuda.stream(side_):
                runner._dense(batches[0])
            stream.wait_stream(side_)
            torch.cuda.synchronize()
            barrier()
            with torch.cuda.graph(kg):
                runner._dense(batches[0])
            torch.cuda.synchronize()
            us_graph = time_k7(lambda i: kg.replay())
            del kg
        except Exception as e:  # report the eager number alone
            print(f"rank {rank}: K7 graph timing unavailable: {e}", file=sys.stderr, flush=True)
        us = us_graph if us_graph is not None else us_eager
        nvl_peak = 770.0
        achieved = egress / (us * 1e-6) / 1e9
        roof = {"kernel": f"K7 dense exchange ({runner.dense_exchange}, split {w})",
                "bound": "nvlink", "achieved": achieved, "peak": nvl_peak, "unit": "GB/s",
                "frac": achieved / nvl_peak, "traffic": None, "algorithmic_bytes": egress,
                "bytes_rule": how, "launch_us": us, "eager_us": us_eager,
                "timing": "graph replay of the exchange alone (all ranks released together, "
                          "max over ranks, median of 10)" if us_graph is not None else "eager",
                "peak_src": "fallback: measured peer copy 770 GB/s per direction (B200_PROFILING.md)",
                # every rank storing to its peer at once (tools/nvlink_bidir.py, N = 2,
                # profiles/r2_n2_k7_studies.txt): the rate both link directions sustain
                "frac_of_bidir_measured": achieved / 680.0,
                "step_share": us / (t_dev / args.steps * 1e6)}

    _mark("kernel timing / roofline done")
    # ---- e2e through the public API: pinned host inputs -> step -> result to host
    pinned = []
    for b in host:
        pinned.append({k: ((torch.from_numpy(v[0]).pin_memory(), torch.from_numpy(v[1]).pin_memory())
                           if isinstance(v, tuple) else torch.from_numpy(v).pin_memory())
                       for k, v in b.items()})
    static = to_dev(host[0])
    e2e_graph = runner.capture(static) if use_graph else None
    res_host = torch.empty(len(wl.tables) or 1, 4, dtype=torch.float32).pin_memory()
    h2d = sum(x.numel() * x.element_size() for v in pinned[0].values()
              for x in (v if isinstance(v, tuple) else (v,)))
    d2h = res_host.numel() * 4

    # the step's host->device copies spread over HP_E2E_STREAMS copy streams
    # (largest tensors first, round robin), joined before the step
    n_cs = int(os.environ.get("HP_E2E_STREAMS", "1"))
    cstreams = [torch.cuda.Stream(device=dev) for _ in range(n_cs)] if n_cs > 1 else []

    def e2e_step(i):
        src = pinned[i % R]
        pairs = []
        for k, v in src.items():
            if isinstance(v, tuple):
                pairs += [(static[k][0], v[0]), (static[k][1], v[1])]
            else:
                pairs.append((static[k], v))
        if cstreams:
            cur = torch.cuda.current_stream()
            pairs.sort(key=lambda p: -p[1].numel() * p[1].element_size())
            for j, (d, s) in enumerate(pairs):
                cs = cstreams[j % n_cs]
                if j < n_cs:
                    cs.wait_stream(cur)
                with torch.cuda.stream(cs):
                    d.copy_(s, non_blocking=True)
            for cs in cstreams[:len(pairs)]:
                cur.wait_stream(cs)
        else:
            for d, s in pairs:
                d.copy_(s, non_blocking=True)
        if e2e_graph:
            e2e_graph.replay()
        else:
            runner.step(static, timed=False)
        if wl.tables:
            for j, t in enumerate(wl.tables):
                res_host[j].copy_(runner.outputs[t.name][0, :4], non_blocking=True)
        torch.cuda.current_stream().synchronize()

    for i in range(2):
        e2e_step(i)
    barrier()
    torch.cuda.synchronize()
    ke = max(5, min(args.steps, 30))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for i in range(ke):
        e2e_step(i)
    b.record(stream)
    torch.cuda.synchronize()
    t_e2e = max_over_ranks(a.elapsed_time(b) / 1e3)
    e2e_value = ups * ke / t_e2e

    _mark("e2e done")
    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        _, dt = time_cpu(wl, 1, args.cpu_steps)
        v = ups / dt
        cpu = {"value": v, "unit": unit, "cores": cpu_threads(), "kind": "port",
               "sample": f"{args.cpu_steps} full oracle steps (1 worker, C restatement, "
                         f"OpenMP x{cpu_threads()}), {dt*1e3:.1f} ms/step"}

    if rank == 0:
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_dev / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (Zipf(1.1) ids, normal grads, hash-initialised tables)",
            "config": config(args, wl) | {"rotations": R, "cuda_graph": bool(graphs),
                                          "steps_per_graph": G,
                                          "exchange": runner.exchange,
                                          "dense_exchange": runner.dense_exchange,
                                          "dense_split": runner.dense_weights or "uniform"}
                      | ({"dense_in": "bf16"} if args.dense_in == "bf16" else {}),
            "e2e": {"value": e2e_value, "unit": unit, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": ke},
            "gpu_launches": launches_per_step * args.steps,
            "launches_per_step": launches_per_step,
            "roofline": roof, "kernels_us": kern, "cpu_baseline": cpu,
            "sparse_exchange": sparse_x,
            "clocks": clk.summary(),
        }
        if check is not None:
            line["parity_check"] = check
        print(json.dumps(line), flush=True)
    # release captured graphs (they reference NCCL and peer windows) before teardown
    graphs = e2e_graph = multis = None
    torch.cuda.synchronize()
    runner.check_errors(sync=True)  # any device error bit of the run raises here
    _mark("errors checked")
    if world > 1:
        errs = runner.exchange_status()
        if any(errs.values()):
            print(f"rank {rank}: exchange error bits {errs}", file=sys.stderr, flush=True)
        barrier()
        torch.cuda.synchronize()
        _mark("teardown")
        # The line is printed and every rank is past the last collective: leave
        # without the NCCL / IPC teardown (measured: a torchrun bench could sit
        # in it until killed; the OS releases the GPU resources of the process)
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)


if __name__ == "__main__":
    main()
