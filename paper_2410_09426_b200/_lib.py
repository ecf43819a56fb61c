"""Thin ctypes binding of libflatquant.so (include/flatquant.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels behind the
C ABI.  torch is used for device memory and streams.  There is no CPU fallback: if the
library is missing or a call fails, a RuntimeError is raised.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libflatquant.so")
# FQ_TRACE_LIB=1 loads the instrumented build (device timelines; profiling scripts only)
if os.environ.get("FQ_TRACE_LIB") == "1":
    LIB_PATH = os.path.join(HERE, "libflatquant_trace.so")
# FQ_LIB=<path>: an experiment build (paper_2410_09426_b200.build.build_variant); testing aid only
if os.environ.get("FQ_LIB"):
    LIB_PATH = os.environ["FQ_LIB"]

FQ_OK, FQ_EINVAL, FQ_ESHAPE, FQ_ENOTSUP, FQ_ECUDA, FQ_ESINGULAR = 0, 1, 2, 3, 4, 5
FQ_F16, FQ_BF16 = 0, 1
FQ_SYM, FQ_ASYM = 0, 1

_c = ctypes
_vp, _i32, _i64, _f32, _u64 = _c.c_void_p, _c.c_int32, _c.c_int64, _c.c_float, _c.c_uint64

# name -> (restype, argtypes); mirrors include/flatquant.h
SIGNATURES = {
    "fq_transform_quant": (_i32, [_vp, _i32, _i64, _i64, _i32, _i32, _vp, _vp, _f32, _i32, _vp, _vp, _vp, _vp]),
    "fq_transform_f32": (_i32, [_vp, _i32, _i64, _i64, _i32, _i32, _vp, _vp, _f32, _vp, _vp, _vp, _vp]),
    "fq_w4a4_linear": (_i32, [_vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _i32, _vp, _i32, _vp]),
    "fq_w4a4_gemm_i32": (_i32, [_vp, _i64, _i32, _vp, _i32, _vp, _vp]),
    "fq_weight_colsum": (_i32, [_vp, _i32, _i32, _vp, _vp]),
    "fq_flatquant_linear": (_i32, [_vp, _i32, _i64, _i32, _i32, _vp, _vp, _f32, _vp, _vp, _i32, _vp, _i32,
                                   _vp, _vp, _vp]),
    "fq_flatquant_linear_host": (_i32, [_vp, _vp, _i32, _i64, _i32, _i32, _vp, _vp, _f32, _vp, _vp, _i32, _vp,
                                        _vp, _i32, _vp, _vp, _vp]),
    "fq_flatquant_linear_host_async": (_i32, [_vp, _vp, _i32, _i64, _i32, _i32, _vp, _vp, _f32, _vp, _vp, _i32, _vp,
                                        _vp, _i32, _vp, _vp, _vp]),
    "fq_prepare_weight": (_i32, [_vp, _i32, _i32, _i64, _i32, _i32, _vp, _vp, _f32, _vp, _vp, _vp, _vp, _u64,
                                 _vp]),
    "fq_prepare_weight_workspace_size": (_u64, [_i32, _i32]),
    "fq_kv_quant": (_i32, [_vp, _i32, _i64, _i64, _i32, _vp, _f32, _vp, _vp, _vp, _vp]),
    "fq_choose_decomposition": (_i32, [_i64, _c.POINTER(_i32), _c.POINTER(_i32)]),
    "fq_set_gemm_impl": (_i32, [_i32]),
    "fq_set_tq_impl": (_i32, [_i32]),
    "fq_launch_count": (_u64, []),
    "fq_status_string": (_c.c_char_p, [_i32]),
    "fq_abi_version": (_i32, []),
    "fq_last_cuda_error": (_i32, []),
}

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load libflatquant.so (fails loudly if it has not been built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"{LIB_PATH} not found: build it with `python -m paper_2410_09426_b200.build` "
                                   "(or __graft_entry__.build()); there is no CPU fallback")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                f = getattr(lib, name)
                f.restype = res
                f.argtypes = args
            _lib = lib
    return _lib


class FlatQuantError(RuntimeError):
    def __init__(self, fn: str, status: int):
        lib = load()
        msg = lib.fq_status_string(status).decode()
        if status == FQ_ECUDA:
            msg += f" (cudaError {lib.fq_last_cuda_error()})"
        super().__init__(f"{fn}: {msg}")
        self.status = status


def check(fn: str, status: int) -> None:
    if status != FQ_OK:
        raise FlatQuantError(fn, status)
