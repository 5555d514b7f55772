import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
# The one-GPU emulated multi-rank tests (test_gpu_emulated.py) keep several
# ranks' spinning exchange waits in flight at once; a lazily loaded kernel's
# first launch synchronises the context and would wait on them (measured:
# every wait times out on the first step). Load modules eagerly, before the
# first CUDA call of the test process.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
# ... and give the emulated ranks' streams distinct hardware queues
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

REF_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def reference():
    """The reference package imported read-only (build container only)."""
    if not REF_SRC.exists():
        pytest.skip("reference not present (GPU box): golden vectors cover this")
    sys.dont_write_bytecode = True
    if str(REF_SRC) not in sys.path:
        sys.path.append(str(REF_SRC))
    import sparseplan

    return sparseplan


@pytest.fixture(scope="session")
def golden():
    import json

    return json.loads((ROOT / "tests" / "golden" / "planner_golden.json").read_text())


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1808_02621_b200 import _lib

    _lib.load()
    return torch.device("cuda:0")
