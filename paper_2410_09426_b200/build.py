"""Build libflatquant.so (all CUDA sources, sm_100a) in-tree with nvcc.

Every .cu is compiled to an object in parallel (objects are cached under build/ by a digest of
the source, the shared headers and the flags, so an edit recompiles only what it touches), then
the objects are linked into one shared library.

Usage: python -m paper_2410_09426_b200.build [-v] [-f] [--trace]
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libflatquant.so")
TRACE_LIB = os.path.join(HERE, "libflatquant_trace.so")
OBJ_DIR = os.path.join(ROOT, "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))) \
        + [os.path.join(ROOT, "include", "flatquant.h")]


def _hash(paths, extra: str) -> str:
    """content digest, independent of where the repo lives (the snapshot runs from another path)"""
    h = hashlib.sha256()
    for f in paths:
        h.update(open(f, "rb").read())
    h.update(extra.replace(ROOT, "<root>").encode())
    return h.hexdigest()


def _digest() -> str:
    return _hash(sources() + _headers(), " ".join(NVCC_FLAGS))


def _compile(src: str, defs: list[str]) -> tuple[str, str]:
    key = _hash([src] + _headers(), " ".join(NVCC_FLAGS + defs))[:16]
    obj = os.path.join(OBJ_DIR, f"{os.path.basename(src)[:-3]}-{key}.o")
    if os.path.exists(obj):
        return obj, ""
    tmp = obj + f".tmp{os.getpid()}"
    r = subprocess.run([NVCC] + NVCC_FLAGS + defs + ["-c", "-o", tmp, src], capture_output=True, text=True)
    log = f"$ nvcc -c {os.path.basename(src)}\n" + r.stdout + r.stderr
    if r.returncode != 0:
        raise RuntimeError(log)
    os.replace(tmp, obj)
    return obj, log


def build_variant(name: str, defines: list[str], only: list[str]) -> str:
    """Experiment build (never loaded by the product): libflatquant_<name>.so with `defines`
    applied to the sources named in `only`; load it with FQ_LIB=<path>."""
    os.makedirs(OBJ_DIR, exist_ok=True)
    objs = []
    for src in sources():
        defs = defines if os.path.basename(src) in only else []
        objs.append(_compile(src, defs)[0])
    lib = os.path.join(HERE, f"libflatquant_{name}.so")
    r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib] + objs,
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stdout + r.stderr)
    return lib


def build(verbose: bool = False, force: bool = False, trace: bool = False) -> str:
    """Build libflatquant.so; trace=True builds the instrumented libflatquant_trace.so instead
    (-DFQ_TRACE: device timelines for scripts/trace_*.py; never loaded by the product)."""
    lib = TRACE_LIB if trace else LIB
    stamp = lib + ".sha256"
    dig = _digest() + ("-trace" if trace else "")
    if not force and os.path.exists(lib) and os.path.exists(stamp) and open(stamp).read() == dig:
        return lib
    os.makedirs(OBJ_DIR, exist_ok=True)
    defs = ["-DFQ_TRACE"] if trace else []
    if force:
        for src in sources():
            key = _hash([src] + _headers(), " ".join(NVCC_FLAGS + defs))[:16]
            p = os.path.join(OBJ_DIR, f"{os.path.basename(src)[:-3]}-{key}.o")
            if os.path.exists(p):
                os.remove(p)
    logs = []
    try:
        with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
            results = list(ex.map(lambda s: _compile(s, defs), sources()))
    except RuntimeError as e:
        with open(os.path.join(HERE, "build_trace.log" if trace else "build.log"), "w") as f:
            f.write(str(e))
        sys.stderr.write(str(e))
        raise RuntimeError(f"nvcc failed building {os.path.basename(lib)} (see paper_2410_09426_b200/build*.log)")
    objs = [o for o, _ in results]
    logs = [lg for _, lg in results]
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib] + objs
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = "\n".join(logs) + " ".join(cmd) + "\n" + r.stdout + r.stderr
    with open(os.path.join(HERE, "build_trace.log" if trace else "build.log"), "w") as f:
        f.write(log)
    if r.returncode != 0:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed linking {os.path.basename(lib)} (see paper_2410_09426_b200/build*.log)")
    if verbose:
        sys.stderr.write(log)
    with open(stamp, "w") as f:
        f.write(dig)
    _prune()
    return lib


def _prune() -> None:
    """drop cached objects of older source versions (keep the current plain and trace builds)"""
    keep = set()
    for src in sources():
        for defs in ([], ["-DFQ_TRACE"]):
            key = _hash([src] + _headers(), " ".join(NVCC_FLAGS + defs))[:16]
            keep.add(f"{os.path.basename(src)[:-3]}-{key}.o")
    for f in glob.glob(os.path.join(OBJ_DIR, "*.o")):
        if os.path.basename(f) not in keep:
            os.remove(f)


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, trace="--trace" in sys.argv))
