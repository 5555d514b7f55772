"""SURVEY §8f rank 2 at N > 1: HybridLM on every GPU of the box (one rank per
GPU) — the forward pulls rows from their owners over NVLink
(HybridRunner.pull / hp_xchg_pull), the backward's IndexedSlices and the dense
LSTM gradient go through the multi-GPU hybrid step. Each rank trains on its own
fixed batch: its loss must fall, and the replicated LSTM must stay identical
on every rank (the dense mean is the same everywhere).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tests/dist_lm_check.py
"""

import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1808_02621_b200 as hp  # noqa: E402
from paper_1808_02621_b200.lm import HybridLM  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = hp.Comm.from_torch_distributed()
    lm = HybridLM(V=50_000, D=128, hidden=256, batch=16, seq=10, samples=512, partitions=8,
                  device=dev, seed=3, rank=rank, world_size=world, comm=comm)
    toks, samp = lm.batch_ids()
    losses = [lm.step(toks, samp) for _ in range(8)]
    torch.cuda.synchronize()
    ok = bool(np.all(np.isfinite(losses)) and losses[-1] < losses[0])
    # the replicated dense Weight stays bit-identical across ranks
    flat = torch.cat([p.detach().reshape(-1) for p in lm.dense_params])
    ref = flat.clone()
    dist.broadcast(ref, 0)
    same = bool(torch.equal(flat, ref))
    lm.runner.check_errors(sync=True)
    print(f"DIST_LM rank {rank}/{world}: {'PASS' if ok and same else 'FAIL'} "
          f"loss {losses[0]:.4f} -> {losses[-1]:.4f} replicas_equal={same}", flush=True)
    flag = torch.tensor([0 if ok and same else 1], device=dev)
    dist.all_reduce(flag)
    lm.runner.close()
    comm.close()
    dist.destroy_process_group()
    sys.exit(int(flag.item() > 0))


if __name__ == "__main__":
    main()
