"""In-tree build of libaxb_b200.so for sm_100a (no GPU needed: nvcc cross-compiles).

    python -m paper_2408_05444_b200.build
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SOURCES = ["axb_iter.cu", "axb_gemm.cu", "axb_solver.cu", "axb_analysis.cu"]
OUT = os.path.join(PKG, "libaxb_b200.so")
# -DAXB_CHECKED: device bounds checks at the iteration kernels' indexing sites
# (the sanitizer substitute; AXB_LIB_VARIANT=checked loads it)
OUT_CHECKED = os.path.join(PKG, "libaxb_b200_checked.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-I", os.path.join(ROOT, "include"),
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_rebuild(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(ROOT, "include", "axb_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    out = OUT_CHECKED if checked else OUT
    if not force and not needs_rebuild(out):
        return out
    tmp = out + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, *(["-DAXB_CHECKED"] if checked else []), "-shared", "-o", tmp,
           *[os.path.join(CSRC, s) for s in SOURCES], "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))
