"""Build libconebp_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2104_13248_b200.build [--force]

The library is compiled from csrc/capi.cu (+ bp_kernels.cuh) with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` and a static CUDA
runtime, so the shared object only needs the NVIDIA driver at run time.
Device code is built with -fmad=false (no contraction of separately rounded
products and sums into FMA, including the packed f32x2 forms); host code without
FMA contraction (-ffp-contract=off): the slab
planner reproduces the kernels' float32 corner arithmetic on the CPU.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
LIB = HERE / "libconebp_b200.so"
SOURCES = [CSRC / "capi.cu", CSRC / "bp_kernels.cuh", CSRC / "fwd_kernels.cuh", CSRC / "fdk.cuh", HERE.parent / "include" / "conebp_b200.h"]

NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-gencode",
    "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    # never contract a*b+c: ptxas fuses packed mul.rn.f32x2 + add.rn.f32x2 into FFMA2
    # unless told not to, which would break bit-exactness with the reference
    "-fmad=false",
    "-Xcompiler",
    "-fPIC,-ffp-contract=off",
    "-shared",
    "-cudart",
    "static",
    "-Xlinker",
    "-rpath,/usr/local/cuda/lib64",
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build libconebp_b200.so")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(src.stat().st_mtime > t for src in SOURCES)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    extra = os.environ.get("CBP_NVCC_EXTRA", "").split()  # tuning experiments, e.g. -DCBP_ZRUN=16
    cmd = [nvcc_path(), *NVCC_FLAGS, *extra, "-o", str(tmp), str(CSRC / "capi.cu")]
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    out = build(force="--force" in sys.argv, verbose=True)
    print(out)
