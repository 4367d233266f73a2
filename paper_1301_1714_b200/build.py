"""Build libdem.so (the CUDA path, sm_100a) in-tree.

    python -m paper_1301_1714_b200.build [--force]

nvcc -gencode arch=compute_100a,code=sm_100a: tcgen05-era B200 target; the
kernels are scalar FP32/FP64 SIMT and integer work (no dense contraction on
this path), so no tensor-core instructions are expected in SASS.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libdem.so")
# the same sources with the ablation kernels (the paper's thread-per-particle
# mapping, half lists, one lane per particle) compiled in: tests and
# `bench.py --sweep` load it for those flags; the product library has none
LIB_ABLATIONS = os.path.join(HERE, "libdem_ablations.so")
SOURCES = [os.path.join(CSRC, f) for f in ("dem_kernels.cu", "dem_api.cu")]
HEADERS = [os.path.join(CSRC, "dem_internal.h"), os.path.join(INCLUDE, "dem.h")]

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-warn-spills",
    "-diag-suppress", "186",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile libdem.so (or, for tuning experiments, a variant `out` with -D defines)."""
    target = out or LIB
    if not force and out is None and not stale():
        return LIB
    if out is None and target == LIB and "DEM_ABLATIONS=1" not in defines:
        build_ablations(force)
    tmp = target + f".tmp{os.getpid()}"
    cmd = [nvcc(), *NVCC_FLAGS, *(f"-D{d}" for d in defines), "-I", INCLUDE, "-I", CSRC,
           *SOURCES, "-o", tmp]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, target)
    return target


def build_ablations(force: bool = False, verbose: bool = False) -> str:
    if force or stale(LIB_ABLATIONS):
        build(force=True, verbose=verbose, out=LIB_ABLATIONS, defines=("DEM_ABLATIONS=1",))
    return LIB_ABLATIONS


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
