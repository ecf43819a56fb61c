"""Pins of the float64 oracle against things other than itself (CPU only).

Each test names what fixes the expected value: a value printed in PAPER.md /
SPEC.md (tests/golden/paper_values.json), an explicit library construction
(np.kron), a closed form, an invariant, or brute force on tiny inputs.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


# ---------------------------------------------------------------- transform a1-a3
@pytest.mark.parametrize("n1,n2", [(a, b) for a in range(1, 9) for b in range(1, 9)])
def test_kron_factored_equals_explicit_kronecker_matrix(n1, n2):
    """vec(V)(P1 (x) P2) = vec(P1^T V P2); explicit n x n matrix via np.kron."""
    g = np.random.default_rng(n1 * 100 + n2)
    x = g.standard_normal((5, n1 * n2))
    p1 = g.standard_normal((n1, n1))
    p2 = g.standard_normal((n2, n2))
    y = O.kron_transform(x, p1, p2)
    ref = x @ np.kron(p1, p2)
    assert np.allclose(y, ref, rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))


def test_column_major_reading_is_rejected():
    """Negative control for reading R1: column-major vec does NOT satisfy the identity,
    so an oracle built on it would fail the explicit-Kronecker pin above."""
    g = np.random.default_rng(7)
    n1, n2 = 3, 4
    v = g.standard_normal((n1, n2))
    p1 = g.standard_normal((n1, n1))
    p2 = g.standard_normal((n2, n2))
    col = (v.flatten(order="F") @ np.kron(p1, p2))
    assert not np.allclose(col, (p1.T @ v @ p2).flatten(order="F"))
    assert np.allclose(v.flatten(order="C") @ np.kron(p1, p2), (p1.T @ v @ p2).flatten(order="C"))


def test_kron_scalar_golden():
    for case in GOLD["kron_scalar"]:
        n1, n2 = case["n1"], case["n2"]
        x = np.arange(2 * n1 * n2, dtype=np.float64).reshape(2, n1 * n2) - 3.0
        y = O.kron_transform(x, case["p1_scale"] * np.eye(n1), case["p2_scale"] * np.eye(n2))
        assert np.array_equal(y, case["factor"] * x)


def test_kron_identity_and_permutation_closed_form():
    x = synth.activations(4, 64, seed=3).astype(np.float64)
    assert np.array_equal(O.kron_transform(x, np.eye(8), np.eye(8)), x)
    p1 = synth.permutation(8, seed=1)
    p2 = synth.permutation(8, seed=2)
    # P = P1 (x) P2 is itself a permutation matrix: y = x P permutes the columns.
    perm = np.kron(p1, p2).argmax(axis=0)          # column j of P has its 1 in row perm[j]
    assert np.array_equal(O.kron_transform(x, p1, p2), x[:, perm])


def test_hadamard_spike_spreads_to_all_codes_7():
    """Sylvester H_{n1} (x) H_{n2} = H_n (normalised), so a spike a e_j maps to |y| = a/sqrt(n)
    everywhere and every code is +-7 at alpha = 1."""
    n1, n2 = 16, 32
    h1, h2 = synth.hadamard(n1), synth.hadamard(n2)
    assert np.allclose(np.kron(h1, h2), synth.hadamard(n1 * n2), atol=1e-15)
    x = np.zeros((3, n1 * n2))
    x[0, 5] = 3.0
    x[1, 511] = -100.0
    x[2, 200] = 1e-3
    q, s, y = O.transform_quant(x, h1, h2, 1.0)
    assert np.allclose(np.abs(y), np.abs(x).max(axis=1, keepdims=True) / math.sqrt(n1 * n2), rtol=1e-12)
    assert np.all(np.abs(q) == 7)


def test_orthogonal_transform_preserves_norm():
    g = np.random.default_rng(11)
    q1, _ = np.linalg.qr(g.standard_normal((16, 16)))
    q2, _ = np.linalg.qr(g.standard_normal((32, 32)))
    x = g.standard_normal((7, 512))
    y = O.kron_transform(x, q1, q2)
    assert np.allclose(np.linalg.norm(y, axis=1), np.linalg.norm(x, axis=1), rtol=1e-12)


def test_mixed_product_property():
    """(P1 (x) P2)(Q1 (x) Q2) = (P1 Q1) (x) (P2 Q2): two transforms == one composed."""
    g = np.random.default_rng(5)
    p1, q1 = g.standard_normal((2, 6, 6))
    p2, q2 = g.standard_normal((2, 10, 10))
    x = g.standard_normal((4, 60))
    two = O.kron_transform(O.kron_transform(x, p1, p2), q1, q2)
    one = O.kron_transform(x, p1 @ q1, p2 @ q2)
    assert np.allclose(two, one, rtol=1e-11, atol=1e-11)


def test_equivalence_before_quantization():
    """X W^T = (X P)(W P^{-T})^T (Eq.3)."""
    n1, n2, N, T = 8, 16, 24, 10
    x = synth.activations(T, n1 * n2, seed=1).astype(np.float64)
    w = synth.weights(N, n1 * n2, seed=1).astype(np.float64)
    p1 = synth.well_conditioned(n1, seed=1, tag="p1").astype(np.float64)
    p2 = synth.well_conditioned(n2, seed=1, tag="p2").astype(np.float64)
    lhs = x @ w.T
    rhs = O.kron_transform(x, p1, p2) @ O.transform_weight(w, p1, p2).T
    assert np.allclose(lhs, rhs, rtol=1e-9, atol=1e-9 * np.abs(lhs).max())
    # weight side equals W P^{-T} with the explicit Kronecker matrix
    P = np.kron(p1, p2)
    assert np.allclose(O.transform_weight(w, p1, p2), w @ np.linalg.inv(P).T, atol=1e-10)


# ---------------------------------------------------------------- quantizer a4-a5
def test_quantizer_golden_examples():
    for case in GOLD["quantizer_examples"]:
        q, s = O.quantize_rows(np.array([case["x"]]), case["clip"])
        assert q.tolist()[0] == case["codes"]
        assert s[0] == pytest.approx(case["scale"], rel=1e-15)


def test_clip_threshold_golden():
    for case in GOLD["clip_threshold"]:
        assert 1.0 / (1.0 + math.exp(-case["theta"])) == pytest.approx(case["alpha"], abs=case["tol"])


def _nearest_grid_bruteforce(y_row, s):
    """Enumerate the 16-point grid {-8..7} s, nearest wins, ties to the even code (R5)."""
    out = []
    for v in y_row:
        best = None
        for c in range(-8, 8):
            d = abs(v - c * s)
            if best is None or d < best[0] - 1e-300 or (d == best[0] and c % 2 == 0):
                best = (d, c)
        out.append(best[1])
    return out


@pytest.mark.parametrize("alpha", [1.0, 0.9, 0.5])
def test_quantizer_matches_bruteforce_grid_search(alpha):
    g = np.random.default_rng(int(alpha * 100))
    y = g.standard_normal((6, 40)) * g.uniform(0.1, 10, size=(6, 1))
    y[2, 3] = 0.0
    q, s = O.quantize_rows(y, alpha)
    for r in range(y.shape[0]):
        assert s[r] == pytest.approx(alpha * np.abs(y[r]).max() / 7, rel=1e-15)
        assert q[r].tolist() == _nearest_grid_bruteforce(y[r], s[r])


def test_quantizer_half_step_bound_and_idempotence():
    """|s q - y| <= s/2 inside the clip range; Q(Q(y)) = Q(y)."""
    x = synth.activations(64, 256, seed=9).astype(np.float64)
    q, s, y = O.transform_quant(x, np.eye(16), np.eye(16), 1.0)
    assert np.array_equal(y, x)
    err = np.abs(O.dequantize_rows(q, s) - y)
    assert np.all(err <= s[:, None] / 2 * (1 + 1e-12))
    q2, s2 = O.quantize_rows(O.dequantize_rows(q, s), 1.0)
    assert np.array_equal(q2, q)
    assert np.allclose(s2, s, rtol=1e-15)


def test_quantizer_zero_row_and_clip_saturation():
    y = np.array([[0.0, 0.0, 0.0, 0.0], [1.0, -1.0, 0.5, -0.25]])
    q, s = O.quantize_rows(y, 0.9)
    assert s[0] == 1.0 and np.all(q[0] == 0)                       # R6
    # alpha = 0.9: max maps to 7/0.9 = 7.78 -> saturates at 7; -max -> -7.78 -> -8
    assert q[1].tolist() == [7, -8, 4, -2]
    with pytest.raises(ValueError):
        O.quantize_rows(y, 0.0)


def test_scale_invariance_of_codes():
    """Codes are invariant to a positive per-row rescale (used by the GPU's exact
    power-of-two prescale); they negate for a negative scalar P away from ties."""
    g = np.random.default_rng(2)
    y = g.standard_normal((5, 64))
    q, s = O.quantize_rows(y)
    q2, s2 = O.quantize_rows(y * 2.0 ** 37)
    assert np.array_equal(q, q2) and np.allclose(s2, s * 2.0 ** 37, rtol=1e-15)
    q3, _ = O.quantize_rows(-y)
    nt = ~O.near_tie_mask(y, s, 1e-9) & (q != -8)
    assert np.array_equal(q3[nt], -q[nt])


# ---------------------------------------------------------------- packing
def test_pack_known_bytes_and_roundtrip():
    assert O.pack_int4(np.array([[1, -1, -8, 7, 0, 0]])).tolist() == [[0xF1, 0x78, 0x00]]
    c = np.array(list(itertools.product(range(-8, 8), repeat=2)), dtype=np.int8).reshape(1, -1)
    assert np.array_equal(O.unpack_int4(O.pack_int4(c)), c)
    with pytest.raises(ValueError):
        O.pack_int4(np.array([[8, 0]]))


# ---------------------------------------------------------------- integer GEMM a6
def test_int_gemm_matches_python_bruteforce():
    qa = synth.random_codes(5, 64, seed=1)
    qw = synth.random_codes(7, 64, seed=2)
    assert np.array_equal(O.int_gemm(qa, qw), O.int_gemm_bruteforce(qa, qw))


def test_int_gemm_matches_int64_numpy_and_extremes():
    qa = synth.random_codes(33, 1024, seed=3)
    qw = synth.random_codes(17, 1024, seed=4)
    assert np.array_equal(O.int_gemm(qa, qw), qa.astype(np.int64) @ qw.astype(np.int64).T)
    K = 28672                                    # largest K in the configs (LLaMA-3-70B down_proj)
    a = np.full((2, K), -8, np.int8)
    b = np.stack([np.full(K, -8, np.int8), np.full(K, 7, np.int8)])
    acc = O.int_gemm(a, b)
    assert acc.tolist() == [[64 * K, -56 * K], [64 * K, -56 * K]]


# ---------------------------------------------------------------- dequant a7 + whole chain
def test_dequant_closed_form():
    acc = np.array([[3, -4], [0, 10]])
    y = O.dequant(acc, [0.5, 2.0], [1.0, 0.25])
    assert y.tolist() == [[1.5, -0.5], [0.0, 5.0]]


def test_whole_chain_within_quantization_error_bound():
    """With P = I, alpha = 1: |x^ - x| <= s_a/2, |w^ - w| <= s_w/2 element-wise, hence
    |Y - X W^T| <= sum_k (|x_k| s_w/2 + |w_k| s_a/2 + s_a s_w/4).  A dropped scale,
    a wrong sign or a transposed operand anywhere in a1-a7 breaks this bound."""
    n1, n2, N, T = 8, 16, 12, 9
    x = synth.activations(T, n1 * n2, seed=4).astype(np.float64)
    w = synth.weights(N, n1 * n2, seed=4).astype(np.float64)
    r = O.flatquant_linear(x, np.eye(n1), np.eye(n2), 1.0, w, 1.0)
    ref = x @ w.T
    sa, sw = r["sa"], r["sw"]
    bound = (np.abs(x).sum(1)[:, None] * sw[None, :] / 2 + np.abs(w).sum(1)[None, :] * sa[:, None] / 2
             + x.shape[1] * sa[:, None] * sw[None, :] / 4)
    assert np.all(np.abs(r["out"] - ref) <= bound * (1 + 1e-12))
    # and it is a real approximation, not trivially satisfied
    assert np.linalg.norm(r["out"] - ref) < 0.2 * np.linalg.norm(ref)


def test_whole_chain_with_transform_approximates_unquantized_product():
    n1, n2, N, T = 16, 32, 64, 16
    x = synth.activations(T, n1 * n2, seed=5, outlier_scale=5.0, pivot_scale=1.0).astype(np.float64)
    w = synth.weights(N, n1 * n2, seed=5).astype(np.float64)
    p1 = synth.well_conditioned(n1, seed=5, tag="p1").astype(np.float64)
    p2 = synth.well_conditioned(n2, seed=5, tag="p2").astype(np.float64)
    r = O.flatquant_linear(x, p1, p2, 1.0, w, 1.0)
    ref = x @ w.T
    assert np.linalg.norm(r["out"] - ref) < 0.35 * np.linalg.norm(ref)


# ---------------------------------------------------------------- decomposition rule
def test_decomposition_golden_and_properties():
    for case in GOLD["decomposition"]:
        assert O.choose_decomposition(case["n"]) == (case["n1"], case["n2"])
    assert O.choose_decomposition(4096) == (64, 64)            # perfect square -> sqrt
    assert O.choose_decomposition(14336) == (112, 128)
    assert O.choose_decomposition(28672) == (128, 224)
    assert O.choose_decomposition(11008) == (86, 128)          # not the paper's 64x172 (R9)
    assert O.choose_decomposition(13) == (1, 13)               # prime
    for n in range(1, 600):
        n1, n2 = O.choose_decomposition(n)
        assert n1 * n2 == n and n1 <= n2
        # no divisor pair strictly between (n1, n2) and the square root
        assert all(n % d for d in range(n1 + 1, math.isqrt(n) + 1))


def test_near_tie_mask():
    y = np.array([[0.5, 0.255, 1.0, -0.75]])
    s = np.array([0.5])
    m = O.near_tie_mask(y, s, 0.02)
    assert m.tolist() == [[False, True, False, True]]


# ---------------------------------------------------------------- asymmetric mode (NEXT-1, R19)
def test_asym_worked_examples():
    """SPEC.md:135 asymmetric min-max with R19's zero-inclusive range.
    [0, 1.5, 3] -> s = 3/15 = 0.2, z = 0, codes [0, 8 (rint(7.5) = 8, half-even), 15];
    [-1, 0.5, 2] -> s = 3/15, z = rint(5) = 5, codes [0, rint(2.5) + 5 = 7, 15];
    one-signed rows keep 0 in the range: [2, 3, 4] -> s = 4/15, z = 0, codes [8, 11, 15];
    [-4, -3, -2] -> z = 15, codes [0, rint(-11.25) + 15 = 4, rint(-7.5) + 15 = 7]."""
    q, s, z = O.quantize_rows_asym(np.array([[0.0, 1.5, 3.0]]))
    assert np.isclose(s[0], 0.2) and z[0] == 0 and q[0].tolist() == [0, 8, 15]
    q, s, z = O.quantize_rows_asym(np.array([[-1.0, 0.5, 2.0]]))
    assert np.isclose(s[0], 0.2) and z[0] == 5 and q[0].tolist() == [0, 7, 15]
    # one-signed rows still include 0 in the range: z stays in [0, 15]
    q, s, z = O.quantize_rows_asym(np.array([[2.0, 3.0, 4.0], [-4.0, -3.0, -2.0], [0.0, 0.0, 0.0]]))
    assert z.tolist() == [0, 15, 0] and s[2] == 1.0 and np.all(q[2] == 0)
    assert q[0].tolist() == [8, 11, 15] and q[1].tolist() == [0, 4, 7]


def test_asym_bruteforce_grid_and_half_step():
    """Codes are the nearest point of the 16-point grid {s (q - z)} (brute force over the grid),
    within s/2 inside the (clipped) range, and the extreme of the range is hit exactly."""
    g = np.random.default_rng(11)
    y = g.standard_normal((40, 48)) * g.uniform(0.1, 50, size=(40, 1)) + g.normal(0, 3, size=(40, 1))
    for alpha in (1.0, 0.85):
        q, s, z = O.quantize_rows_asym(y, alpha)
        grid = (np.arange(16)[None, :] - z[:, None]) * s[:, None]              # [R, 16]
        best = np.abs(y[:, :, None] - grid[:, None, :]).argmin(axis=2)
        dist_q = np.abs(y - O.dequantize_rows_asym(q, s, z))
        dist_b = np.abs(y - np.take_along_axis(grid, best, 1))
        assert np.allclose(dist_q, dist_b, atol=1e-12)                        # nearest grid point
        hi = np.maximum(alpha * y.max(1), 0)
        lo = np.minimum(alpha * y.min(1), 0)
        inside = (y <= hi[:, None] + 1e-12) & (y >= lo[:, None] - 1e-12)
        assert np.all(dist_q[inside] <= s.repeat(48).reshape(40, 48)[inside] / 2 + 1e-12)
        assert np.all((z >= 0) & (z <= 15)) and np.all((q >= 0) & (q <= 15))


def test_asym_linear_equals_dequantized_product():
    """w4a4_linear_asym is exactly deq(A) deq(W)^T (closed form), and equals the symmetric
    GEMM of the q - 8 codes minus the (z - 8) colsum(W) correction the GPU epilogue applies."""
    g = np.random.default_rng(4)
    x = g.standard_normal((9, 64)); w = g.standard_normal((7, 64))
    qa, sa, za = O.quantize_rows_asym(x, 0.9)
    qw, sw = O.quantize_rows(w)
    y = O.w4a4_linear_asym(qa, sa, za, qw, sw)
    ref = O.dequantize_rows_asym(qa, sa, za) @ O.dequantize_rows(qw, sw).T
    assert np.allclose(y, ref, rtol=1e-12, atol=1e-12)
    acc8 = O.int_gemm(qa.astype(np.int64) - 8, qw)
    corr = (za - 8)[:, None] * qw.astype(np.int64).sum(1)[None, :]
    assert np.array_equal(acc8 - corr, O.int_gemm(qa.astype(np.int64) - za[:, None], qw))


# ---------------------------------------------------------------- KV cache (NEXT-3, R20)
def test_kv_quant_worked_example():
    """PAPER.md:293 (keys transformed head by head, row vector times P_h) + R19's quantizer.
    Non-symmetric P_h = [[1, 2], [3, 4]] so that P_h vs P_h^T is caught:
    k = [1, 0] -> y = [1, 2]: s = 2/15, z = 0, codes [rint(7.5) = 8, 15];
    k = [0, -1] -> y = [-3, -4]: s = 4/15, z = 15, codes [rint(-11.25) + 15 = 4, 0]."""
    q, s, z, y = O.kv_quant(np.array([[1.0, 0.0], [0.0, -1.0]]), np.array([[1.0, 2.0], [3.0, 4.0]]))
    assert y.tolist() == [[1.0, 2.0], [-3.0, -4.0]]
    assert np.allclose(s, [2 / 15, 4 / 15]) and z.tolist() == [0, 15]
    assert q.tolist() == [[8, 15], [4, 0]]


def test_kv_quant_orthogonal_roundtrip_bound():
    """With an orthogonal P_h (q and k are both rotated, q k^T = (q P_h)(k P_h)^T),
    dequantizing and undoing the rotation recovers each head vector within the quantizer's half
    step: ||deq(k P_h) P_h^T - k||_2 <= sqrt(D) s / 2 per head vector (alpha = 1, no clipping),
    and the attention logits of a rotated query move by at most ||q||_2 sqrt(D) s / 2."""
    g = np.random.default_rng(3)
    for D in (64, 128):
        ph, _ = np.linalg.qr(g.standard_normal((D, D)))
        k = g.standard_normal((50, D)) * g.uniform(0.1, 20, size=(50, 1))
        q, s, z, _ = O.kv_quant(k, ph, 1.0)
        rec = O.dequantize_rows_asym(q, s, z) @ ph.T
        err = np.linalg.norm(rec - k, axis=1)
        assert np.all(err <= np.sqrt(D) * s / 2 + 1e-9)
        qry = g.standard_normal((3, D))
        logits = (qry @ ph) @ O.dequantize_rows_asym(q, s, z).T
        bound = np.linalg.norm(qry, axis=1)[:, None] * (np.sqrt(D) * s / 2)[None, :]
        assert np.all(np.abs(logits - qry @ k.T) <= bound + 1e-9)


def test_kv_quant_is_unit_kronecker():
    """A head vector transform is the Kronecker transform with n1 = 1 (P = [1] (x) P_h):
    kv_quant equals transform_quant_asym with p1 = [[1]]: identical codes and zero points, scales
    and transformed values equal up to float64 summation order."""
    g = np.random.default_rng(8)
    kv = g.standard_normal((33, 64))
    ph = g.standard_normal((64, 64))
    a = O.kv_quant(kv, ph, 0.9)
    b = O.transform_quant_asym(kv, np.ones((1, 1)), ph, 0.9)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[2], b[2])
    assert np.allclose(a[1], b[1], rtol=1e-12, atol=0) and np.allclose(a[3], b[3], rtol=1e-12, atol=1e-12)
