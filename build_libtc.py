"""Builds libtc.so in-tree for sm_100a (B200) with nvcc.

    python build_libtc.py [-v]

The shared library lands in the package directory (paper_1801_03855_b200/libtc.so) so it travels to
the GPU box with the repository snapshot.  cudart is linked statically and libcuda is not
linked at all (driver entry points are resolved at run time), so the library also loads on a
machine without a GPU driver.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.abspath(__file__))
HERE = os.path.join(ROOT, "paper_1801_03855_b200")
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtc.so")
SOURCES = ["tc_plan.cpp", "tc_runtime.cu", "tc_symmem.cu", "tc_kernels.cu",
           "tc_kernels_allreduce.cu", "tc_kernels_sgd.cu", "tc_kernels_easgd.cu",
           "tc_kernels_esgd.cu", "tc_kernels_bcast.cu", "tc_kernels_easync.cu"]
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
    deps = [os.path.join(CSRC, s) for s in SOURCES + ["tc_internal.h", "tc_kernels.cuh"]]
    deps.append(os.path.join(ROOT, "include", "tc.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, ptxas_info: bool = False,
          out: str = LIB, defines: tuple = ()) -> str:
    """Compiles the sources in parallel (one nvcc per file) and links them.  `out`/`defines`
    build experimental variants (e.g. -DTC_LD_MODE=1) next to the product library."""
    if not force and out == LIB and not _stale():
        return out
    tmp = tempfile.mkdtemp(prefix="libtc_")
    extra = (["-Xptxas", "-v"] if ptxas_info else []) + [f"-D{d}" for d in defines]
    objs, procs = [], []
    for s in SOURCES:
        obj = os.path.join(tmp, s + ".o")
        cmd = [NVCC] + FLAGS + extra + ["-c", os.path.join(CSRC, s), "-o", obj]
        cmd.remove("-shared")
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                          text=True)))
        objs.append(obj)
    failed = False
    for s, pr in procs:
        so, se = pr.communicate()
        if verbose or pr.returncode != 0:
            sys.stdout.write(so)
            sys.stderr.write(se)
        failed |= pr.returncode != 0
    if failed:
        shutil.rmtree(tmp, ignore_errors=True)
        raise RuntimeError("nvcc failed")
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
            "-Xcompiler", "-fPIC,-fvisibility=hidden"] + objs + ["-o", out + ".tmp"]
    r = subprocess.run(link, capture_output=True, text=True)
    shutil.rmtree(tmp, ignore_errors=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc link failed ({r.returncode})")
    os.replace(out + ".tmp", out)
    return out


PROBE_SRC = os.path.join(ROOT, "tools", "nvl_probe.cu")
PROBE_LIB = os.path.join(ROOT, "tools", "bin", "libnvl_probe.so")


def build_probe(force: bool = False) -> str:
    """tools/nvl_probe.cu -> tools/bin/libnvl_probe.so: the all-peer copy kernels bench.py runs
    beside the step as the same-run P2P ceiling; not part of libtc."""
    if not force and os.path.exists(PROBE_LIB) and \
            os.path.getmtime(PROBE_LIB) >= os.path.getmtime(PROBE_SRC):
        return PROBE_LIB
    os.makedirs(os.path.dirname(PROBE_LIB), exist_ok=True)
    subprocess.check_call([NVCC, "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-shared", "-Xcompiler", "-fPIC", "-o", PROBE_LIB, PROBE_SRC])
    return PROBE_LIB


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--out", default=LIB)
    ap.add_argument("-D", action="append", default=[], dest="defines")
    a = ap.parse_args()
    build(verbose=a.v, force=True, ptxas_info=a.v, out=os.path.abspath(a.out),
          defines=tuple(a.defines))
