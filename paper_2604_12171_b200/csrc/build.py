"""Build libpipelive.so in-tree for sm_100a with nvcc (no torch extension, no JIT cache).

Usage: python -m paper_2604_12171_b200.csrc.build  [--force]
The .so lands next to the package (paper_2604_12171_b200/libpipelive.so) so it
travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
PKG = HERE.parent
ROOT = PKG.parent
OUT = PKG / "libpipelive.so"
SOURCES = ["vmm.cu", "store.cu", "patch.cu", "ipc.cu", "kernels.cu", "attn.cu", "verify.cu", "exact.cu", "act.cu", "abi.cu"]
HEADERS = ["internal.h", "common.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-I", str(ROOT / "include"),
]

# exact.cu: no fma contraction beyond the explicit __fma_rn calls (bit-exact vs the oracle)
EXTRA = {"exact.cu": ["-fmad=false"]}


def _stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = [HERE / f for f in SOURCES + HEADERS] + [ROOT / "include" / "pipelive.h", Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return OUT
    objdir = HERE / "_obj"
    objdir.mkdir(exist_ok=True)
    objs = []
    hdr_t = max((HERE / h).stat().st_mtime for h in HEADERS)
    hdr_t = max(hdr_t, (ROOT / "include" / "pipelive.h").stat().st_mtime, Path(__file__).stat().st_mtime)
    jobs = []
    for src in SOURCES:
        obj = objdir / (src + ".o")
        objs.append(str(obj))
        if not force and obj.exists() and obj.stat().st_mtime > max(hdr_t, (HERE / src).stat().st_mtime):
            continue
        cmd = [NVCC, *FLAGS, *EXTRA.get(src, []), "-c", str(HERE / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        jobs.append(cmd)
    # translation units are independent: compile them concurrently
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for r in list(ex.map(lambda c: subprocess.run(c, check=True), jobs)):
            pass
    # export only the C-ABI: pl_* symbols are marked default-visibility below
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs,
           "-o", str(OUT), "--cudart", "static"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
