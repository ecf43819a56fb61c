"""Build libflatquant.so (all CUDA sources, sm_100a) in-tree with nvcc.

Usage: python -m paper_2410_09426_b200.build [-v]
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libflatquant.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v", "-shared",
    "-I", os.path.join(ROOT, "include"),
]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _digest() -> str:
    h = hashlib.sha256()
    for f in sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))) \
            + [os.path.join(ROOT, "include", "flatquant.h")]:
        h.update(open(f, "rb").read())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


TRACE_LIB = os.path.join(HERE, "libflatquant_trace.so")


def build(verbose: bool = False, force: bool = False, trace: bool = False) -> str:
    """Build libflatquant.so; trace=True builds the instrumented libflatquant_trace.so instead
    (-DFQ_TRACE: device timelines for scripts/trace_tq.py; never loaded by the product)."""
    lib = TRACE_LIB if trace else LIB
    stamp = lib + ".sha256"
    dig = _digest() + ("-trace" if trace else "")
    if not force and os.path.exists(lib) and os.path.exists(stamp) and open(stamp).read() == dig:
        return lib
    cmd = [NVCC] + NVCC_FLAGS + (["-DFQ_TRACE"] if trace else []) + ["-o", lib] + sources()
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = r.stdout + r.stderr
    with open(os.path.join(HERE, "build_trace.log" if trace else "build.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + log)
    if r.returncode != 0:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed building {os.path.basename(lib)} (see paper_2410_09426_b200/build*.log)")
    if verbose:
        sys.stderr.write(log)
    with open(stamp, "w") as f:
        f.write(dig)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, trace="--trace" in sys.argv))
