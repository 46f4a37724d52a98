"""Builds libtc.so in-tree for sm_100a (B200) with nvcc.

    python build_libtc.py [-v]

The shared library lands in the package directory (paper_1801_03855_b200/libtc.so) so it travels to
the GPU box with the repository snapshot.  cudart is linked statically and libcuda is not
linked at all (driver entry points are resolved at run time), so the library also loads on a
machine without a GPU driver.
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
HERE = os.path.join(ROOT, "paper_1801_03855_b200")
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtc.so")
SOURCES = ["tc_plan.cpp", "tc_runtime.cu", "tc_symmem.cu", "tc_kernels.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-std=c++17", "-O3", "-lineinfo", "--expt-relaxed-constexpr", "-diag-suppress", "177",
    "-gencode", "arch=compute_100a,code=sm_100a",
    # parity-critical arithmetic: no FMA contraction, no flush-to-zero, IEEE div/sqrt (R5)
    "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared", "-cudart", "static",
    "-I", os.path.join(ROOT, "include"),
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + ["tc_internal.h"]]
    deps.append(os.path.join(ROOT, "include", "tc.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, ptxas_info: bool = False) -> str:
    if not force and not _stale():
        return LIB
    cmd = [NVCC] + FLAGS + (["-Xptxas", "-v"] if ptxas_info else []) + \
        [os.path.join(CSRC, s) for s in SOURCES] + ["-o", LIB + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stdout.write(r.stdout)
        sys.stderr.write(r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({r.returncode})")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force=True, ptxas_info="-v" in sys.argv)
