"""Build the fp64 oracle shared library (TEST INFRASTRUCTURE, not product code).

Building the checker is not using it: ``__graft_entry__.build()`` compiles it so
the tests and ``bench.py --impl reference`` can load it; the product path never
does.
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "dem_oracle.cpp")
LIB = os.path.join(HERE, "libdem_oracle.so")

# -ffp-contract=off: no a*b+c contraction, so the fp64 predicate and overlap are
# the exact expressions DESIGN.md reading R14 defines. -march is left generic so
# the library built here also runs on the GPU box's host.
FLAGS = ["-O2", "-std=c++17", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["g++", *FLAGS, SRC, "-o", tmp])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
