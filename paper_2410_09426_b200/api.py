"""Python face of the C ABI: the same entry points as include/flatquant.h, taking torch tensors.

Marshalling only (pointers, sizes, dtypes, the current CUDA stream); the work runs in the CUDA
kernels of libflatquant.so.  Allocating conveniences (`transform_quant`, `w4a4_linear`, ...)
create outputs with torch and then call the same entry points.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import FQ_BF16, FQ_F16, FQ_SYM, check, load

__all__ = [
    "fq_transform_quant", "fq_transform_f32", "fq_w4a4_linear", "fq_w4a4_gemm_i32", "fq_flatquant_linear",
    "fq_weight_colsum", "weight_colsum", "transform_quant_asym", "fq_kv_quant", "kv_quant", "fq_prepare_weight",
    "fq_flatquant_linear_host", "fq_choose_decomposition", "fq_set_gemm_impl", "fq_set_tq_impl", "fq_launch_count",
    "fq_abi_version", "transform_quant", "transform_f32", "w4a4_linear", "w4a4_gemm_i32", "prepare_weight",
    "flatquant_linear",
]


def _ptr(t):
    return None if t is None else t.data_ptr()     # the argtypes are c_void_p (_lib.py)


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(stream) -> int:
    """the cudaStream_t handle: `stream`, else the current stream of the current device (read
    without building a torch.cuda.Stream object: a decode-size call is otherwise host-bound)"""
    if stream is not None:
        return stream.cuda_stream
    if _raw_stream is not None:
        return _raw_stream(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def _fq_dtype(dt: torch.dtype) -> int:
    if dt == torch.float16:
        return FQ_F16
    if dt == torch.bfloat16:
        return FQ_BF16
    raise TypeError(f"unsupported dtype {dt} (fp16 or bf16)")


def _cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("all tensors must be CUDA tensors (there is no CPU path)")


def _need(cond, msg):
    if not cond:
        raise ValueError(msg)


def _buf(t, name, shape, dtype):
    """An output/parameter buffer the C ABI addresses as a dense row-major array of `shape`."""
    if t is None:
        return
    # messages are formatted only on failure (this runs for every buffer of every call)
    if t.shape != shape:
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.dtype != dtype:
        raise ValueError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _rows(x, name, min_cols):
    """A [rows, >= min_cols] matrix with unit column stride (the row stride is passed)."""
    if not (x.dim() == 2 and x.stride(1) == 1):
        raise ValueError(f"{name} must be 2-D with unit column stride")
    if x.shape[1] < min_cols:
        raise ValueError(f"{name}: {x.shape[1]} columns < {min_cols}")


# ------------------------------------------------------------------ raw entry points
def _tq_args(x, n1, n2, p1, p2, q, scale, zero=None):
    _rows(x, "x", n1 * n2)
    T = x.shape[0]
    _buf(p1, "p1", (n1, n1), x.dtype)
    _buf(p2, "p2", (n2, n2), x.dtype)
    _buf(q, "q", (T, n1 * n2 // 2), torch.uint8)
    _buf(scale, "scale", (T,), torch.float32)
    _buf(zero, "zero", (T,), torch.int8)


def fq_transform_quant(x, n1, n2, p1, p2, alpha, q, scale, zero=None, qmode=FQ_SYM, stream=None):
    _cuda(x, p1, p2, q, scale, zero)
    _tq_args(x, n1, n2, p1, p2, q, scale, zero)
    st = load().fq_transform_quant(_ptr(x), _fq_dtype(x.dtype), x.shape[0], x.stride(0), n1, n2, _ptr(p1),
                                   _ptr(p2), float(alpha), qmode, _ptr(q), _ptr(scale), _ptr(zero), _stream(stream))
    check("fq_transform_quant", st)


def fq_transform_f32(x, n1, n2, p1, p2, alpha, q, scale, y, stream=None):
    _cuda(x, p1, p2, q, scale, y)
    _tq_args(x, n1, n2, p1, p2, q, scale)
    _buf(y, "y", (x.shape[0], n1 * n2), torch.float32)
    st = load().fq_transform_f32(_ptr(x), _fq_dtype(x.dtype), x.shape[0], x.stride(0), n1, n2, _ptr(p1), _ptr(p2),
                                 float(alpha), _ptr(q), _ptr(scale), _ptr(y), _stream(stream))
    check("fq_transform_f32", st)


def _gemm_args(qa, qw, K):
    _need(qa.dim() == 2 and qw.dim() == 2, "qa and qw must be 2-D")
    K = qa.shape[1] * 2 if K is None else K
    _buf(qa, "qa", (qa.shape[0], K // 2), torch.uint8)
    _buf(qw, "qw", (qw.shape[0], K // 2), torch.uint8)
    return K


def fq_w4a4_linear(qa, sa, qw, sw, y, K=None, za=None, colsum_w=None, stream=None):
    _cuda(qa, sa, qw, sw, y, za, colsum_w)
    K = _gemm_args(qa, qw, K)
    T, N = qa.shape[0], qw.shape[0]
    _buf(sa, "sa", (T,), torch.float32)
    _buf(sw, "sw", (N,), torch.float32)
    _buf(za, "za", (T,), torch.int8)
    _buf(colsum_w, "colsum_w", (N,), torch.int32)
    _need(y.dtype in (torch.float16, torch.bfloat16), "y must be fp16 or bf16")
    _buf(y, "y", (T, N), y.dtype)
    st = load().fq_w4a4_linear(_ptr(qa), _ptr(sa), _ptr(za), qa.shape[0], K, _ptr(qw), _ptr(sw), _ptr(colsum_w),
                               qw.shape[0], _ptr(y), _fq_dtype(y.dtype), _stream(stream))
    check("fq_w4a4_linear", st)


def fq_w4a4_gemm_i32(qa, qw, acc, K=None, stream=None):
    _cuda(qa, qw, acc)
    K = _gemm_args(qa, qw, K)
    _buf(acc, "acc", (qa.shape[0], qw.shape[0]), torch.int32)
    st = load().fq_w4a4_gemm_i32(_ptr(qa), qa.shape[0], K, _ptr(qw), qw.shape[0], _ptr(acc), _stream(stream))
    check("fq_w4a4_gemm_i32", st)


def fq_weight_colsum(qw, colsum, K=None, stream=None):
    _cuda(qw, colsum)
    _need(qw.dim() == 2, "qw must be 2-D")
    K = qw.shape[1] * 2 if K is None else K
    _buf(qw, "qw", (qw.shape[0], K // 2), torch.uint8)
    _buf(colsum, "colsum", (qw.shape[0],), torch.int32)
    check("fq_weight_colsum", load().fq_weight_colsum(_ptr(qw), qw.shape[0], K, _ptr(colsum), _stream(stream)))


def fq_kv_quant(kv, p_h, alpha, q, scale, zero, stream=None):
    """kv [R, D] (row stride kv.stride(0)), p_h [D, D]; outputs q [R, D/2], scale [R], zero [R]."""
    _cuda(kv, p_h, q, scale, zero)
    _need(kv.dim() == 2 and kv.stride(1) == 1, "kv must be 2-D with unit column stride")
    R, D = kv.shape
    _buf(p_h, "p_h", (D, D), kv.dtype)
    _buf(q, "q", (R, D // 2), torch.uint8)
    _buf(scale, "scale", (R,), torch.float32)
    _buf(zero, "zero", (R,), torch.int8)
    st = load().fq_kv_quant(_ptr(kv), _fq_dtype(kv.dtype), kv.shape[0], kv.stride(0), kv.shape[1], _ptr(p_h),
                            float(alpha), _ptr(q), _ptr(scale), _ptr(zero), _stream(stream))
    check("fq_kv_quant", st)


def kv_quant(kv, p_h, alpha=1.0, stream=None):
    """KV-cache quantization: returns (q packed [R, D/2] holding q - 8,
    scale [R], zero [R] int8 holding z - 8) of kv_r P_h, one asymmetric group per head vector."""
    R, D = kv.shape
    q = torch.empty((R, D // 2), dtype=torch.uint8, device=kv.device)
    s = torch.empty((R,), dtype=torch.float32, device=kv.device)
    z = torch.empty((R,), dtype=torch.int8, device=kv.device)
    fq_kv_quant(kv, p_h, alpha, q, s, z, stream=stream)
    return q, s, z


def _linear_args(x, n1, n2, p1, p2, qw, sw, y, q_ws, s_ws):
    # the C entry point takes x as a dense [T, n1 n2] matrix (row stride n1 n2)
    _need(x.dim() == 2 and x.shape[1] == n1 * n2 and x.is_contiguous(), "x must be a contiguous [T, n1*n2] matrix")
    _tq_args(x, n1, n2, p1, p2, q_ws, s_ws)
    _need(qw.dim() == 2, "qw must be 2-D")
    _buf(qw, "qw", (qw.shape[0], n1 * n2 // 2), torch.uint8)
    _buf(sw, "sw", (qw.shape[0],), torch.float32)
    _need(y.dtype in (torch.float16, torch.bfloat16), "y must be fp16 or bf16")
    _buf(y, "y", (x.shape[0], qw.shape[0]), y.dtype)


def fq_flatquant_linear(x, n1, n2, p1, p2, alpha, qw, sw, y, q_ws, s_ws, stream=None):
    _cuda(x, p1, p2, qw, sw, y, q_ws, s_ws)
    _linear_args(x, n1, n2, p1, p2, qw, sw, y, q_ws, s_ws)
    st = load().fq_flatquant_linear(_ptr(x), _fq_dtype(x.dtype), x.shape[0], n1, n2, _ptr(p1), _ptr(p2),
                                    float(alpha), _ptr(qw), _ptr(sw), qw.shape[0], _ptr(y), _fq_dtype(y.dtype),
                                    _ptr(q_ws), _ptr(s_ws), _stream(stream))
    check("fq_flatquant_linear", st)


def fq_flatquant_linear_host(x_host, x_dev, n1, n2, p1, p2, alpha, qw, sw, y_host, y_dev, q_ws, s_ws, stream=None,
                             sync=True):
    """x_host / y_host are CPU tensors (pinned recommended).  sync=True synchronises the stream
    (fq_flatquant_linear_host); sync=False only enqueues (fq_flatquant_linear_host_async)."""
    _cuda(x_dev, p1, p2, qw, sw, y_dev, q_ws, s_ws)
    if x_host.is_cuda or y_host.is_cuda:
        raise ValueError("x_host and y_host must be host tensors")
    _linear_args(x_dev, n1, n2, p1, p2, qw, sw, y_dev, q_ws, s_ws)
    _buf(x_host, "x_host", tuple(x_dev.shape), x_dev.dtype)
    _buf(y_host, "y_host", tuple(y_dev.shape), y_dev.dtype)
    name = "fq_flatquant_linear_host" if sync else "fq_flatquant_linear_host_async"
    st = getattr(load(), name)(_ptr(x_host), _ptr(x_dev), _fq_dtype(x_dev.dtype), x_dev.shape[0], n1, n2,
                               _ptr(p1), _ptr(p2), float(alpha), _ptr(qw), _ptr(sw), qw.shape[0],
                               _ptr(y_host), _ptr(y_dev), _fq_dtype(y_dev.dtype), _ptr(q_ws), _ptr(s_ws),
                               _stream(stream))
    check(name, st)


def fq_choose_decomposition(n: int) -> tuple[int, int]:
    a, b = ctypes.c_int32(), ctypes.c_int32()
    check("fq_choose_decomposition", load().fq_choose_decomposition(int(n), ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def fq_set_gemm_impl(impl: int) -> None:
    check("fq_set_gemm_impl", load().fq_set_gemm_impl(int(impl)))


def fq_set_tq_impl(impl: int) -> None:
    check("fq_set_tq_impl", load().fq_set_tq_impl(int(impl)))


def fq_launch_count() -> int:
    return int(load().fq_launch_count())


def fq_abi_version() -> int:
    return int(load().fq_abi_version())


# ------------------------------------------------------------------ allocating conveniences
def transform_quant(x, n1, n2, p1, p2, alpha=1.0, stream=None):
    T = x.shape[0]
    q = torch.empty((T, n1 * n2 // 2), dtype=torch.uint8, device=x.device)
    s = torch.empty((T,), dtype=torch.float32, device=x.device)
    fq_transform_quant(x, n1, n2, p1, p2, alpha, q, s, stream=stream)
    return q, s


def transform_quant_asym(x, n1, n2, p1, p2, alpha=1.0, stream=None):
    """FQ_ASYM: returns (q packed [T, n/2] holding q - 8, scale [T], zero [T]
    int8 holding z - 8)."""
    T = x.shape[0]
    q = torch.empty((T, n1 * n2 // 2), dtype=torch.uint8, device=x.device)
    s = torch.empty((T,), dtype=torch.float32, device=x.device)
    z = torch.empty((T,), dtype=torch.int8, device=x.device)
    fq_transform_quant(x, n1, n2, p1, p2, alpha, q, s, zero=z, qmode=_lib.FQ_ASYM, stream=stream)
    return q, s, z


def weight_colsum(qw, stream=None):
    colsum = torch.empty((qw.shape[0],), dtype=torch.int32, device=qw.device)
    fq_weight_colsum(qw, colsum, stream=stream)
    return colsum


def transform_f32(x, n1, n2, p1, p2, alpha=1.0, stream=None):
    T = x.shape[0]
    q = torch.empty((T, n1 * n2 // 2), dtype=torch.uint8, device=x.device)
    s = torch.empty((T,), dtype=torch.float32, device=x.device)
    y = torch.empty((T, n1 * n2), dtype=torch.float32, device=x.device)
    fq_transform_f32(x, n1, n2, p1, p2, alpha, q, s, y, stream=stream)
    return q, s, y


def w4a4_linear(qa, sa, qw, sw, out_dtype=torch.float16, za=None, colsum_w=None, stream=None):
    y = torch.empty((qa.shape[0], qw.shape[0]), dtype=out_dtype, device=qa.device)
    fq_w4a4_linear(qa, sa, qw, sw, y, za=za, colsum_w=colsum_w, stream=stream)
    return y


def w4a4_gemm_i32(qa, qw, stream=None):
    acc = torch.empty((qa.shape[0], qw.shape[0]), dtype=torch.int32, device=qa.device)
    fq_w4a4_gemm_i32(qa, qw, acc, stream=stream)
    return acc


def fq_prepare_weight(w, n1, n2, p1, p2, alpha_w, qw, sw, colsum_w=None, workspace=None, stream=None):
    """Raw entry point (synchronous, see include/flatquant.h); allocates the workspace if not given."""
    _cuda(w, p1, p2, qw, sw, colsum_w)
    _tq_args(w, n1, n2, p1, p2, qw, sw)
    _buf(colsum_w, "colsum_w", (w.shape[0],), torch.int32)
    lib = load()
    need = int(lib.fq_prepare_weight_workspace_size(n1, n2))
    if workspace is None:
        workspace = torch.empty((max(need, 1),), dtype=torch.uint8, device=w.device)
    st = lib.fq_prepare_weight(_ptr(w), _fq_dtype(w.dtype), w.shape[0], w.stride(0), n1, n2, _ptr(p1), _ptr(p2),
                               float(alpha_w), _ptr(qw), _ptr(sw), _ptr(colsum_w), _ptr(workspace),
                               workspace.numel() * workspace.element_size(), _stream(stream))
    check("fq_prepare_weight", st)


def prepare_weight(w, n1, n2, p1, p2, alpha_w=1.0, with_colsum=False, stream=None):
    """Offline weight side of Eq.3: W'_o = P1^{-1} W~_o P2^{-T}, quantized per
    output channel, entirely on the GPU through fq_prepare_weight: float64
    Gauss-Jordan inverses, then the activation kernel with (P1^{-T}, P2^{-T}, alpha_w).
    Returns (qw [N, K/2] uint8, sw [N] fp32) or, with_colsum, also colsum_w [N] int32."""
    N = w.shape[0]
    qw = torch.empty((N, n1 * n2 // 2), dtype=torch.uint8, device=w.device)
    sw = torch.empty((N,), dtype=torch.float32, device=w.device)
    cs = torch.empty((N,), dtype=torch.int32, device=w.device) if with_colsum else None
    fq_prepare_weight(w, n1, n2, p1, p2, alpha_w, qw, sw, colsum_w=cs, stream=stream)
    return (qw, sw, cs) if with_colsum else (qw, sw)


def flatquant_linear(x, n1, n2, p1, p2, alpha, qw, sw, out_dtype=torch.float16, stream=None):
    """Whole hot path for one linear: returns Y [T, N]."""
    T = x.shape[0]
    y = torch.empty((T, qw.shape[0]), dtype=out_dtype, device=x.device)
    q_ws = torch.empty((T, n1 * n2 // 2), dtype=torch.uint8, device=x.device)
    s_ws = torch.empty((T,), dtype=torch.float32, device=x.device)
    fq_flatquant_linear(x, n1, n2, p1, p2, alpha, qw, sw, y, q_ws, s_ws, stream=stream)
    return y
