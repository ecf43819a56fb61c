"""FlatQuant online hot path -- float64 CPU ORACLE.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product path (``paper_2410_09426_b200``) never imports it and
shares no code with it.

What it computes, each function citing the
passage of ``PAPER.md`` (arXiv 2410.09426) it follows:

  a1-a3  y_t = vec_row(P1^T . reshape(x_t, n1, n2) . P2)        Eq.3
  a4     s_t = alpha . max|y_t| / 7   (s_t = 1 for an all-zero token)
                                          Eq.1; PAPER.md:258-259, 367
  a5     q   = clamp(rint(y / s_t), -8, 7), packed two nibbles per byte
  a6     acc[t,o] = sum_k q_a[t,k] q_w[o,k]   (exact integer)
  a7     Y[t,o]  = acc[t,o] . s_a[t] . s_w[o]                  PAPER.md:88 (Y = X W^T)

plus the offline weight side W'_o = P1^{-1} . reshape(W_o) . P2^{-T}
(Eq.3 weight factor) quantized per output channel
(PAPER.md:367-368).

Readings of the paper (all listed in DESIGN.md §"Readings"):
  R1  vec() is row-major (C order): the only order for which
      vec(V)(P1 (x) P2) = vec(P1^T V P2) holds.
  R2  the kernel computes P1^T X P2; PAPER.md:314's
      "P1 X P2" is a typo.
  R3  symmetric per-token activations / per-channel weights,
      signed grid [-8, 7], step s = alpha . max|y| / 7 (Eq.1 writes the unsigned
      set {0..2^b-1}; for symmetric quantization the signed grid is used).
  R4  alpha in (0, 1] scales the absmax AFTER the transform;
      values beyond +-alpha.max saturate at the code bounds.
  R5  round-half-to-even (the paper is silent).
  R6  an all-zero token gets s = 1 and codes 0 (the paper is silent).
  R7  nibble packing: element 2i in the low nibble of byte i, two's complement
      (the paper is silent; CUTLASS/QuaRot convention).
  R8  inputs are the fp16/bf16 values the GPU sees, widened exactly to float64.

Every function is float64 (or exact integer) throughout.  Parity pins:
tests/test_oracle.py (explicit Kronecker matrix, closed forms, brute force).
No function here is "parity unpinned"; see DESIGN.md §"Oracle pins".
"""
from __future__ import annotations

import numpy as np

QMIN, QMAX = -8, 7          # signed 4-bit grid (R3)
QDIV = 7.0                  # 2^(b-1) - 1 for b = 4 (R3)


def _f64(a) -> np.ndarray:
    """Widen fp16/bf16/fp32 input to float64 exactly (R8)."""
    return np.asarray(a).astype(np.float64)


# ---------------------------------------------------------------------------
# A7: decomposition rule, §3.1 "we select n1*, n2* = argmin(n1+n2)
# s.t. n1 n2 = n and n1 <= n2"
# ---------------------------------------------------------------------------
def choose_decomposition(n: int) -> tuple[int, int]:
    if n < 1:
        raise ValueError("n must be >= 1")
    best = None
    for n1 in range(1, n + 1):
        if n % n1:
            continue
        n2 = n // n1
        if n1 > n2:
            break
        if best is None or n1 + n2 < best[0] + best[1]:
            best = (n1, n2)
    return best


# ---------------------------------------------------------------------------
# a1-a3: Kronecker transform, Eq.3:
#   Q(X P) with P = P1 (x) P2  ==  Q(P1^T x_1 X~ x_2 P2),  X~ in R^{k x n1 x n2}
# ---------------------------------------------------------------------------
def kron_transform(x, p1, p2) -> np.ndarray:
    """y_t = vec_row(P1^T . V_t . P2) with V_t = x_t.reshape(n1, n2) (R1, R2)."""
    x = _f64(x)
    p1 = _f64(p1)
    p2 = _f64(p2)
    n1, n2 = p1.shape[0], p2.shape[0]
    if p1.shape != (n1, n1) or p2.shape != (n2, n2):
        raise ValueError("P1, P2 must be square")
    if x.ndim != 2 or x.shape[1] != n1 * n2:
        raise ValueError("x must be [T, n1*n2]")
    T = x.shape[0]
    v = x.reshape(T, n1, n2)                 # X~
    y = np.matmul(np.matmul(p1.T[None, :, :], v), p2[None, :, :])   # P1^T V P2
    return y.reshape(T, n1 * n2)


def kron_matrix(p1, p2) -> np.ndarray:
    """The full n x n matrix P = P1 (x) P2; for small-shape pins only."""
    return np.kron(_f64(p1), _f64(p2))


# ---------------------------------------------------------------------------
# a4-a5: per-row symmetric INT4 quantizer, Eq.1 with the
# per-token (activations) / per-channel (weights) granularity of PAPER.md:367
# and the clipping ratio alpha of PAPER.md:258-259.
# ---------------------------------------------------------------------------
def _round(v: np.ndarray, rounding: str) -> np.ndarray:
    if rounding == "half_even":                       # R5
        return np.rint(v)
    if rounding == "half_away":                       # SPEC.md:176 alternative
        return np.sign(v) * np.floor(np.abs(v) + 0.5)
    raise ValueError(rounding)


def quantize_rows(y, alpha: float = 1.0, rounding: str = "half_even"):
    """Return (codes int8 [R, C], scales float64 [R]) for each row of y.

    s_r = alpha . max_j |y_rj| / 7 (s_r = 1 if the row is all zero, R6);
    q_rj = clamp(round(y_rj / s_r), -8, 7).
    """
    if not (0.0 < alpha <= 1.0):
        raise ValueError("alpha must be in (0, 1]")
    y = _f64(y)
    m = np.max(np.abs(y), axis=1) if y.shape[1] else np.zeros(y.shape[0])
    s = alpha * m / QDIV
    s = np.where(m == 0.0, 1.0, s)
    v = y / s[:, None]
    q = np.clip(_round(v, rounding), QMIN, QMAX).astype(np.int8)
    return q, s


def dequantize_rows(codes, scales) -> np.ndarray:
    return np.asarray(codes, dtype=np.float64) * _f64(scales)[:, None]


# ---------------------------------------------------------------------------
# a4-a5, asymmetric mode (reading R19).  The paper quantizes
# activations per-token symmetric and uses asymmetric min-max quantization for
# the KV cache; SPEC.md:135 defines asymmetric as s = clip (max - min) / (2^b - 1)
# with a zero point on the unsigned grid {0..2^b-1} (Eq.1's Omega(b)).  Reading R19:
# the range is widened to include 0 (lo = min(alpha min y, 0), hi = max(alpha max y, 0)), the
# usual min-max convention, so the zero point is an integer in [0, 15] and zero is exactly
# representable.
#   s = (hi - lo) / 15 (s = 1 if hi == lo, i.e. an all-zero row)   z = rint(-lo / s)
#   q = clamp(rint(y / s) + z, 0, 15)                                dequant: s (q - z)
# ---------------------------------------------------------------------------
AQMAX = 15                                # 2^b - 1 for b = 4


def quantize_rows_asym(y, alpha: float = 1.0, rounding: str = "half_even"):
    """Return (codes int8 in [0, 15] [R, C], scales float64 [R], zero points int64 [R])."""
    if not (0.0 < alpha <= 1.0):
        raise ValueError("alpha must be in (0, 1]")
    y = _f64(y)
    if y.shape[1]:
        hi = np.maximum(alpha * np.max(y, axis=1), 0.0)
        lo = np.minimum(alpha * np.min(y, axis=1), 0.0)
    else:
        hi = lo = np.zeros(y.shape[0])
    s = (hi - lo) / AQMAX
    s = np.where(s == 0.0, 1.0, s)
    z = _round(-lo / s, rounding).astype(np.int64)
    q = np.clip(_round(y / s[:, None], rounding) + z[:, None], 0, AQMAX).astype(np.int8)
    return q, s, z


def dequantize_rows_asym(codes, scales, zeros) -> np.ndarray:
    return (np.asarray(codes, dtype=np.float64) - np.asarray(zeros, np.float64)[:, None]) * _f64(scales)[:, None]


def transform_quant_asym(x, p1, p2, alpha: float = 1.0, rounding: str = "half_even"):
    """Returns (codes int8 [0,15] [T, n], scales float64 [T], zeros int64 [T], y float64 [T, n])."""
    y = kron_transform(x, p1, p2)
    q, s, z = quantize_rows_asym(y, alpha, rounding)
    return q, s, z, y


def w4a4_linear_asym(qa, sa, za, qw, sw) -> np.ndarray:
    """Y[t,o] = s_a[t] s_w[o] sum_k (q_a[t,k] - z_a[t]) q_w[o,k]  (asymmetric activations,
    symmetric weights): the dequantized product, Y = deq(A) deq(W)^T."""
    qa_c = np.asarray(qa, np.int64) - np.asarray(za, np.int64)[:, None]
    return dequant(int_gemm(qa_c, qw), sa, sw)



# ---------------------------------------------------------------------------
# NEXT-3: KV-cache quantization.  PAPER.md:291-297 §3.2: P_h / P_v "transform the key and value
# cache head by head" (P_h a full head_dim x head_dim matrix; P_v is merged into the weights, so
# values are quantized untransformed, i.e. P = I).  PAPER.md:369 §4.1 and 1101-1104 App. "KV
# Cache Quantization": "group-wise asymmetric quantization with the size of 128", which "matches
# the head dimension": one group = one head vector (reading R20).  The asymmetric
# quantizer is R19's (quantize_rows_asym); alpha is the KV clipping threshold.
# ---------------------------------------------------------------------------
def kv_quant(kv, p_h, alpha: float = 1.0, rounding: str = "half_even"):
    """kv [R, D] head vectors (R = tokens x heads), p_h [D, D].  y_r = kv_r P_h (row vector times
    matrix), then per-row asymmetric INT4.  Returns (codes int8 [0,15] [R, D], scales [R],
    zeros int64 [R], y float64 [R, D])."""
    kv = _f64(kv)
    p_h = _f64(p_h)
    if p_h.shape != (kv.shape[1], kv.shape[1]):
        raise ValueError("p_h must be [D, D] with D = kv.shape[1]")
    y = kv @ p_h
    q, s, z = quantize_rows_asym(y, alpha, rounding)
    return q, s, z, y

# ---------------------------------------------------------------------------
# a5: packing (R7): byte i of a row holds element 2i (low nibble) and 2i+1.
# ---------------------------------------------------------------------------
def pack_int4(codes) -> np.ndarray:
    """Signed codes in [-8, 7] -> two's-complement nibbles (asymmetric codes q in [0, 15] are
    packed as q - 8, reading R19)."""
    c = np.asarray(codes, dtype=np.int16)
    if c.shape[-1] % 2:
        raise ValueError("row length must be even")
    if c.min(initial=0) < QMIN or c.max(initial=0) > QMAX:
        raise ValueError("codes out of the 4-bit range")
    u = (c & 0xF).astype(np.uint8)
    return (u[..., 0::2] | (u[..., 1::2] << 4)).astype(np.uint8)


def unpack_int4(packed) -> np.ndarray:
    p = np.asarray(packed, dtype=np.uint8)
    lo = (p & 0xF).astype(np.int16)
    hi = (p >> 4).astype(np.int16)
    lo = np.where(lo >= 8, lo - 16, lo)
    hi = np.where(hi >= 8, hi - 16, hi)
    out = np.empty(p.shape[:-1] + (p.shape[-1] * 2,), dtype=np.int8)
    out[..., 0::2] = lo
    out[..., 1::2] = hi
    return out


# ---------------------------------------------------------------------------
# a1-a5 fused: the north_star's flat_transform_quant(X, P1, P2, clip)
# ---------------------------------------------------------------------------
def transform_quant(x, p1, p2, alpha: float = 1.0, rounding: str = "half_even"):
    """Returns (codes int8 [T, n], scales float64 [T], y float64 [T, n])."""
    y = kron_transform(x, p1, p2)
    q, s = quantize_rows(y, alpha, rounding)
    return q, s, y


# ---------------------------------------------------------------------------
# Offline weight side (Eq.3 weight factor; "the weights P^{-1} W^T
# can be pre-computed offline"):  W'_o = P1^{-1} . W~_o . P2^{-T},
# i.e. W' = W P^{-T}; then per-channel symmetric RTN.
# ---------------------------------------------------------------------------
def transform_weight(w, p1, p2) -> np.ndarray:
    w = _f64(w)
    p1i = np.linalg.inv(_f64(p1))
    p2i = np.linalg.inv(_f64(p2))
    n1, n2 = p1i.shape[0], p2i.shape[0]
    N = w.shape[0]
    wt = w.reshape(N, n1, n2)                                     # W~
    out = np.matmul(np.matmul(p1i[None, :, :], wt), p2i.T[None, :, :])
    return out.reshape(N, n1 * n2)


def prepare_weight(w, p1, p2, alpha_w: float = 1.0, rounding: str = "half_even"):
    """Returns (codes int8 [N, K], scales float64 [N], W' float64 [N, K])."""
    wp = transform_weight(w, p1, p2)
    q, s = quantize_rows(wp, alpha_w, rounding)
    return q, s, wp


# ---------------------------------------------------------------------------
# a6: integer GEMM acc = Q_a Q_w^T (PAPER.md:241 outer product; PAPER.md:315 INT4
# GEMM).  Exact.  The float64 matmul below IS the integer result: every
# product q_a q_w is an integer in [-56, 64] and every partial sum, in any
# order, is an integer of magnitude <= 64 K < 2^53, so no float64 operation
# rounds (pinned against int64 brute force in tests/test_oracle.py).
# ---------------------------------------------------------------------------
def int_gemm(qa, qw) -> np.ndarray:
    qa = np.asarray(qa)
    qw = np.asarray(qw)
    if qa.shape[1] != qw.shape[1]:
        raise ValueError("K mismatch")
    if qa.shape[1] * 64 >= 2 ** 53:
        raise ValueError("K too large for the exact float64 path")
    acc = qa.astype(np.float64) @ qw.astype(np.float64).T
    return acc.astype(np.int64)


def int_gemm_bruteforce(qa, qw) -> np.ndarray:
    """Plain triple loop in Python ints (tiny shapes only)."""
    qa = np.asarray(qa).tolist()
    qw = np.asarray(qw).tolist()
    out = [[sum(a * b for a, b in zip(ra, rb)) for rb in qw] for ra in qa]
    return np.asarray(out, dtype=np.int64).reshape(len(qa), len(qw))


# ---------------------------------------------------------------------------
# a7: dequant epilogue, Y = acc . s_a[t] . s_w[o] (per-token x per-channel)
# ---------------------------------------------------------------------------
def dequant(acc, sa, sw) -> np.ndarray:
    return np.asarray(acc, dtype=np.float64) * _f64(sa)[:, None] * _f64(sw)[None, :]


def w4a4_linear(qa, sa, qw, sw) -> np.ndarray:
    """north_star w4a4_linear(packed A, packed W, scales) on unpacked codes."""
    return dequant(int_gemm(qa, qw), sa, sw)


def flatquant_linear(x, p1, p2, alpha, w, alpha_w=1.0):
    """Whole chain a1-a7 for one linear: returns dict of every intermediate."""
    qa, sa, y = transform_quant(x, p1, p2, alpha)
    qw, sw, wp = prepare_weight(w, p1, p2, alpha_w)
    acc = int_gemm(qa, qw)
    return dict(y=y, qa=qa, sa=sa, qw=qw, sw=sw, wp=wp, acc=acc, out=dequant(acc, sa, sw))


# ---------------------------------------------------------------------------
# Near-tie classification used by the code-parity bar (SURVEY.md §8(c) bar 3):
# v = y/s in code units; a code may differ by +-1 only where v is within tau
# of a rounding boundary (k + 1/2).  (The asymmetric bar's additional clamp
# exemption is applied by the test helper, tests/parity.py:check_asym.)
# ---------------------------------------------------------------------------
def near_tie_mask(y, s, tau: float) -> np.ndarray:
    v = _f64(y) / _f64(s)[:, None]
    frac = np.abs(v - np.floor(v) - 0.5)
    return frac <= tau
