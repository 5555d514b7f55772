"""Multi-GPU parity check of HybridRunner (NCCL path), one rank per GPU.

    python -m torch.distributed.run --standalone --nproc-per-node N tests/dist_gpu_check.py

Every rank recomputes the single-process oracle of the same step for all
ranks' (seeded) batches and checks, bit-exactly, its pulled rows and the
partitions it homes; the dense allreduce is checked within 1e-5 rel + 1e-6 abs.
Prints one "DIST_CHECK rank r: PASS/FAIL ..." line per rank; exit 1 on failure.
"""

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1808_02621_b200 as hp  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1808_02621_b200.synth import TableShape, Workload, make_batch  # noqa: E402


def _split(spec: str, world: int):
    """'auto' | 'uniform' | 'first0' (rank 0 takes no dense reduction chunk)."""
    return [0.0] + [1.0] * (world - 1) if spec == "first0" else spec


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = hp.Comm.from_torch_distributed()
    opt_kind = os.environ.get("HP_CHECK_OPT", "adagrad")
    xmode = os.environ.get("HP_CHECK_XCHG", "p2p")
    dmode = os.environ.get("HP_CHECK_DENSE", xmode)
    from paper_1808_02621_b200 import _lib

    for kv in filter(None, os.environ.get("HP_CHECK_KNOBS", "").split(",")):
        k, v = kv.split("=")
        getattr(_lib.load(), f"hp_debug_set_{k}")(int(v))
    lm1b = os.environ.get("HP_CHECK_SHAPE") == "lm1b"
    if lm1b:  # BASELINE configs[1]: 2 x 800k x 512, T = 2560 / 2560 + 8192, 9.4M dense, P = 8
        from paper_1808_02621_b200.synth import WORKLOADS

        base = WORKLOADS["lm1b"]
        wl = Workload("check_lm1b", base.tables, dict(base.dense),
                      {"kind": opt_kind, "lr": 0.1, "init_acc": 0.1}, 2560, partitions=8)
        parts = {"embedding": 8, "softmax": 8}
    else:
        wl = Workload("check", [TableShape("embedding", 60_000, 128, 2560),
                                TableShape("softmax", 60_000, 256, 2560, sampled=3000)],
                      {"lstm": int(os.environ.get("HP_CHECK_DENSE_ELEMS", "50000"))},
                      {"kind": opt_kind, "lr": 0.1, "init_acc": 0.1}, 2560, partitions=8)
        parts = {"embedding": 8, "softmax": 12}
    graph = hp.load_graph_spec(json.dumps(wl.graph_json()))
    cluster = hp.ClusterSpec.b200_box(world)
    arch = os.environ.get("HP_CHECK_ARCH", "hybrid")
    if arch == "ar":  # SURVEY §8f baselines: every Weight AR / every Weight PS
        plan = hp.transform_ar(graph, cluster)
    elif arch == "ps":
        plan = hp.transform_ps(graph, cluster, local_agg=True, partitions=parts)
    else:
        plan = hp.transform_hybrid(graph, cluster, partitions=parts)
    # HP_CHECK_DENSE_IN=bf16: the dense gradients arrive in bf16 (in_dtype)
    dense_in = torch.bfloat16 if os.environ.get("HP_CHECK_DENSE_IN") == "bf16" else torch.float32
    runner = hp.HybridRunner(plan, graph, cluster, rank=rank, world_size=world, comm=comm,
                             optimizer=hp.OptimizerConfig(kind=opt_kind, lr=0.1), device=dev,
                             seed=5, exchange=xmode, dense_exchange=None if dmode == "default" else dmode,
                             dense_split=_split(os.environ.get("HP_CHECK_SPLIT", "auto"), world),
                             dense_in_dtype=dense_in)
    hpar = {"lr": 0.1, "beta1": 0.9, "beta2": 0.999, "eps": 1e-8}
    empty = os.environ.get("HP_CHECK_EMPTY") == "1"

    def batch_of(step, r):
        """Seeded batch of rank r; with HP_CHECK_EMPTY=1 the last rank sends no
        embedding ids at step 2 (an empty IndexedSlices through the exchange)."""
        b = make_batch(wl, seed=step, rank=r)
        if empty and step == 2 and r == world - 1:
            ids, vals = b["embedding"]
            b["embedding"] = (ids[:0].copy(), vals[:0].copy())
        if dense_in == torch.bfloat16:  # the oracle sees the bf16 values, widened
            b["lstm"] = torch.from_numpy(b["lstm"]).to(torch.bfloat16).float().numpy()
        return b

    names = [v.name for v in graph.variables]
    if lm1b:  # lazily paged full tables, initialised at every row the steps touch
        from oracle import coracle

        touched = {t.name: np.concatenate([batch_of(s, r)[t.name][0] for s in (1, 2, 3, 4)
                                           for r in range(world)]) for t in wl.tables}
        states = {t.name: orc.lazy_state(opt_kind, t.V, t.D, 5 * 1000 + names.index(t.name),
                                         touched[t.name], 0.1) for t in wl.tables}
    else:
        states = {t.name: orc.init_state(opt_kind, t.V, t.D, 5 * 1000 + i + 1, 0.1)
                  for i, t in enumerate(wl.tables)}
    ok, why = True, []

    def oracle_step(name, step, tb):
        if name in runner.ar_tables:
            orc.ar_sparse_step(states[name], opt_kind, hpar, step, tb)
        else:
            V = next(t.V for t in wl.tables if t.name == name)
            (coracle if lm1b else orc).sparse_step(states[name], opt_kind, hpar, step, tb, V,
                                                   plan.partitions_of[name],
                                                   plan.owner_table(name))
    def to_dev(b):
        return {k: ((torch.from_numpy(v[0]).to(dev), torch.from_numpy(v[1]).to(dev))
                    if isinstance(v, tuple) else torch.from_numpy(v).to(dense_in).to(dev))
                for k, v in b.items()}

    staged = {s: to_dev(batch_of(s, rank)) for s in (1, 2, 3)}
    if xmode == "p2p":
        runner.prefetch(staged[1])  # steps 1-3 run pipelined (plan of step s+1 built during s)
    for step in (1, 2, 3):
        batches = [batch_of(step, r) for r in range(world)]
        mine = batches[rank]
        batch = staged[step]
        stats = runner.step(batch, next_batch=staged.get(step + 1) if xmode == "p2p" else None)
        for t in wl.tables:
            oracle_step(t.name, step, [b[t.name] for b in batches])
            got = runner.outputs[t.name].cpu().numpy()
            if not np.array_equal(got, orc.pull_rows(states[t.name]["w"], mine[t.name][0])):
                ok = False
                why.append(f"step {step} {t.name}: pulled rows differ")
            tab = runner.tables[t.name]
            if lm1b:  # the touched rows this rank homes (the oracle's other rows are lazy zeros)
                rows = np.unique(touched[t.name])
                p = np.searchsorted(tab.bounds, rows, side="right") - 1
                sel = tab.part_base_host[p] >= 0
                srow = tab.part_base_host[p[sel]] + rows[sel] - tab.bounds[p[sel]]
                got_w = tab.w[torch.from_numpy(srow).to(dev)].cpu().numpy()
                if not np.array_equal(got_w, states[t.name]["w"][rows[sel]]):
                    ok = False
                    why.append(f"step {step} {t.name} homed touched rows differ")
                continue
            w = tab.w.cpu().numpy()
            for p in tab.owned:
                lo, hi = int(tab.bounds[p]), int(tab.bounds[p + 1])
                b = int(tab.part_base_host[p])
                if not np.array_equal(w[b:b + hi - lo], states[t.name]["w"][lo:hi]):
                    ok = False
                    why.append(f"step {step} {t.name} partition {p} differs")
        ref = orc.dense_allreduce([b["lstm"] for b in batches], 1.0 / world)
        got = runner.dense_out["lstm"][:ref.size].cpu().numpy()
        if not np.allclose(got, ref, rtol=1e-5, atol=1e-6):
            ok = False
            why.append(f"step {step} dense differs (max {np.abs(got - ref).max():.3g})")
        if runner.dense_exchange in ("p2p", "p2p-sm", "p2p-pipe", "p2p-pull") and not runner.dense_ps:  # rank order
            seq = np.zeros_like(batches[0]["lstm"])
            for b in batches:
                seq = seq + b["lstm"]
            if not np.array_equal(got, seq * np.float32(1.0 / world)):
                ok = False
                why.append(f"step {step} p2p dense not bit-exact vs rank-order sum")
        eg, ing = stats.per_machine_bytes.per_machine[rank]
        if world > 1 and not (eg > 0 and ing > 0):
            ok = False
            why.append("no exchange bytes recorded")
    if xmode == "p2p":
        errs = runner.exchange_status()
        if any(errs.values()):
            ok = False
            why.append(f"exchange error bits {errs}")
        # the same step replayed from a CUDA graph must give the same bytes
        if ok:
            step = 4
            batches = [batch_of(step, r) for r in range(world)]
            mine = batches[rank]
            static = to_dev(mine)
            g = runner.capture(static, warmup=1)  # runs step 4 eagerly, records one step
            g.replay()                            # executes step 5
            torch.cuda.synchronize()
            del g  # release the captured NCCL/peer work before tearing the comms down
            for st_ in (4, 5):
                for t in wl.tables:
                    oracle_step(t.name, st_, [b[t.name] for b in batches])
            torch.cuda.synchronize()
            if True:  # Adam's step size comes from the device step counter
                for t in wl.tables:
                    got = runner.outputs[t.name].cpu().numpy()
                    if not np.array_equal(got, orc.pull_rows(states[t.name]["w"], mine[t.name][0])):
                        ok = False
                        why.append(f"graph replay {t.name}: pulled rows differ")
        runner.close()
    print(f"DIST_CHECK rank {rank}/{world} opt={opt_kind} xchg={xmode} dense={runner.dense_exchange} "
          f"shape={'lm1b' if lm1b else 'small'}: "
          f"{'PASS' if ok else 'FAIL'} {why[:4]}", flush=True)
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    failed = int(flag.item() > 0)
    if os.environ.get("HP_CHECK_TEARDOWN", "1") == "1":
        comm.close()
        dist.destroy_process_group()
    print(f"DIST_CHECK rank {rank} exiting", flush=True)
    sys.exit(failed)


if __name__ == "__main__":
    main()
