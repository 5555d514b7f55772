"""Multi-GPU parity (NCCL path) — runs tests/dist_gpu_check.py under torchrun
when the box has >= 2 GPUs (skipped on a 1-GPU box)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _ngpu():
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("opt,xchg,dense,knobs,arch", [
    # BASELINE configs[1] shapes with the default transports (the bench's path)
    ("adagrad", "p2p", "default", "shape=lm1b", "hybrid"),
    ("adagrad", "p2p", "p2p", "", "hybrid"),
    # weighted reduction split (rank 0 takes no chunk), SM stores and copy engines
    ("adagrad", "p2p", "p2p-sm", "split=first0", "hybrid"),
    # bf16 dense gradients (in_dtype): SM stores (bf16 on the links) and NCCL (widened first)
    ("adagrad", "p2p", "p2p-sm", "dense_in=bf16", "hybrid"),
    ("sgd", "p2p", "nccl", "dense_in=bf16", "hybrid"),
    # the split push (short items on a side stream; HP_SPLIT_PUSH=1)
    ("adam", "p2p", "p2p-sm", "split_push=1", "hybrid"),
    # the SM-store dense exchange's scatter by LSU stores (default: TMA bulk copies)
    ("adagrad", "p2p", "p2p-sm", "dar_tma=0", "hybrid"),
    ("sgd", "p2p", "p2p-sm", "dar_rg_tma=24", "hybrid"),
    # the SM-store dense exchange in 2 and 5 buckets (default 1)
    ("adagrad", "p2p", "p2p-sm", "dar_buckets=2", "hybrid"),
    ("sgd", "p2p", "p2p-sm", "dar_buckets=5", "hybrid"),
    # the last rank pushes an empty IndexedSlices for one table at step 2
    ("sgd", "p2p", "nccl", "empty=1", "hybrid"),
    ("sgd", "p2p", "p2p", "split=first0", "hybrid"),
    ("adam", "p2p", "nccl", "", "hybrid"),
    ("adagrad", "p2p", "nvls", "", "hybrid"),
    ("adagrad", "p2p", "p2p-pipe", "", "hybrid"),
    ("adam", "p2p", "p2p-pull", "", "hybrid"),
    # the alternative kernels behind the instrumentation knobs stay parity-checked
    ("adagrad", "p2p", "p2p-sm", "owner_stream=0,rowstream=1,pdl=1", "hybrid"),
    ("sgd", "nccl", "nccl", "", "hybrid"),
    # SURVEY §8f baselines: sparse under AR (AllGatherv), dense under PS (reduce + bcast)
    ("adagrad", "p2p", "p2p", "", "ar"),
    ("adam", "p2p", "p2p", "", "ps")])
def test_multi_gpu_step_matches_oracle(opt, xchg, dense, knobs, arch):
    n = min(_ngpu(), 8)
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    split, empty, shape = "auto", "0", "small"
    if knobs.startswith("shape="):
        shape, knobs = knobs.split("=", 1)[1], ""
    if knobs.startswith("split="):
        split, knobs = knobs.split("=", 1)[1], ""
    if knobs.startswith("empty="):
        empty, knobs = knobs.split("=", 1)[1], ""
    dense_in = "f32"
    if knobs.startswith("dense_in="):
        dense_in, knobs = knobs.split("=", 1)[1], ""
    split_push = "0"
    if knobs.startswith("split_push="):
        split_push, knobs = knobs.split("=", 1)[1], ""
    env = dict(os.environ, HP_CHECK_OPT=opt, HP_CHECK_XCHG=xchg, HP_CHECK_DENSE=dense,
               HP_CHECK_KNOBS=knobs, HP_CHECK_ARCH=arch, HP_CHECK_SPLIT=split,
               HP_CHECK_EMPTY=empty, HP_CHECK_SHAPE=shape, HP_CHECK_DENSE_IN=dense_in,
               HP_SPLIT_PUSH=split_push,
               # the pipelined dense exchange cuts each chunk into 64 KB pieces: many of them
               HP_CHECK_DENSE_ELEMS="1000004" if dense == "p2p-pipe" else "50000")
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
           str(n), "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(ROOT / "tests" / "dist_gpu_check.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    import re

    lines = re.findall(r"DIST_CHECK rank \d+/\d+ [^\n]*?: (PASS|FAIL)", res.stdout)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert len(lines) == n and set(lines) == {"PASS"}, res.stdout[-3000:]


def test_multi_gpu_lm_consumer():
    """HybridLM across the box's GPUs (forward pull from owners over NVLink)."""
    n = min(_ngpu(), 8)
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
           str(n), "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(ROOT / "tests" / "dist_lm_check.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    import re

    # ranks print concurrently: their lines may interleave on one line
    verdicts = re.findall(r"DIST_LM rank \d+/\d+: (PASS|FAIL)", res.stdout)
    assert res.returncode == 0 and len(verdicts) == n and set(verdicts) == {"PASS"}, (
        res.stdout[-3000:] + res.stderr[-3000:])
