"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
entry point declared in include/hybridpath.h (no compute calls here)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    text = (ROOT / "include" / "hybridpath.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hp_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_1808_02621_b200 import _build, _lib

    _build.build()
    return _lib.load()


def test_every_declared_symbol_exported(lib):
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n


def test_binding_covers_header():
    from paper_1808_02621_b200 import _lib

    assert set(_declared()) == set(_lib.symbols())


def test_version_and_errors(lib):
    assert lib.hp_version() == 100
    assert isinstance(lib.hp_last_error(), bytes)


def test_workspace_query_is_host_only(lib):
    small = lib.hp_dedup_ws_bytes(2560, 512, 8, 8)
    big = lib.hp_dedup_ws_bytes(10_000_000, 128, 128, 8)
    assert 0 < small < big


def test_sass_is_sm100a():
    import subprocess

    so = ROOT / "paper_1808_02621_b200" / "lib" / "libhybridpath.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_structs_match_header():
    from paper_1808_02621_b200._lib import Optim, Slab

    assert ctypes.sizeof(Optim) == 9 * 4 + 4 + 8 + 8 + 4 + 4  # + pad, 2 pointers, len, tail pad
    assert ctypes.sizeof(Slab) == 8 * 4 + 8 + 4 + 4
