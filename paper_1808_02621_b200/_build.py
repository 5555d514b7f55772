"""Build libhybridpath.so (sm_100a) in-tree with nvcc.

Used by ``__graft_entry__.build()`` and ``python -m paper_1808_02621_b200._build``.
The library links the pip NCCL that torch itself loads (2.28.x, same soname),
with an rpath so the GPU box (same image) resolves it without LD_LIBRARY_PATH.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libhybridpath.so"
SOURCES = ["capi.cu", "dedup.cu", "reduce.cu", "rows.cu", "comm.cu", "p2p.cu", "nvls.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs() -> tuple[Path, Path]:
    import nvidia.nccl as nccl  # the NCCL torch loads

    base = Path(list(nccl.__path__)[0])
    return base / "include", base / "lib"


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    raise RuntimeError("nvcc not found")


def _compile(src: Path, obj: Path, inc: Path) -> None:
    cmd = [nvcc(), *ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
           "--expt-relaxed-constexpr", "-Xptxas", "-v", f"-I{ROOT / 'include'}", f"-I{inc}",
           "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = obj.with_suffix(".ptxas.txt")
    log.write_text(res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr[-4000:]}")


def build(force: bool = False, verbose: bool = False) -> Path:
    srcs = [CSRC / s for s in SOURCES]
    hdrs = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "hybridpath.h"]
    if LIB.exists() and not force:
        newest = max(p.stat().st_mtime for p in srcs + hdrs)
        if LIB.stat().st_mtime >= newest:
            return LIB
    inc, libd = nccl_dirs()
    obj_dir = PKG / "build"
    obj_dir.mkdir(exist_ok=True)
    LIBDIR.mkdir(exist_ok=True)
    objs = [obj_dir / (s.stem + ".o") for s in srcs]
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        list(ex.map(lambda so: _compile(so[0], so[1], inc), zip(srcs, objs)))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), f"-L{libd}",
           "-l:libnccl.so.2", f"-Xlinker=-rpath={libd}"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
    os.replace(tmp, LIB)
    if verbose:
        for o in objs:
            print(o.with_suffix(".ptxas.txt").read_text())
    return LIB


if __name__ == "__main__":
    path = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(path)
