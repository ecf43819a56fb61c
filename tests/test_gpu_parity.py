"""GPU parity: the CUDA path (called through the C ABI) against the float64 oracle.

Small cases run element by element; the BASELINE configs run at full size on the GPU in the
launch configuration bench.py uses, compared on sampled tokens (first 256, which include the
pivot token 0, plus 256 random ones) that the oracle recomputes one by one.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from tests import parity

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2410_09426_b200 as fq
    DEV = torch.device("cuda:0")


def to_dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(DEV)


def np_of(t):
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        t = t.float()
    return t.numpy()


def make_inputs(T, n1, n2, seed=0, tdtype=torch.float16, **kw):
    x = torch.from_numpy(synth.activations(T, n1 * n2, seed=seed, dtype=np.float32, **kw)).to(tdtype)
    p1 = torch.from_numpy(synth.well_conditioned(n1, seed=seed, tag="p1", dtype=np.float32)).to(tdtype)
    p2 = torch.from_numpy(synth.well_conditioned(n2, seed=seed, tag="p2", dtype=np.float32)).to(tdtype)
    return x, p1, p2


def run_tq(x, p1, p2, alpha, n1, n2):
    q, s, y = fq.transform_f32(x.to(DEV), n1, n2, p1.to(DEV), p2.to(DEV), alpha)
    torch.cuda.synchronize()
    return np_of(q), np_of(s), np_of(y)


SHAPES = [(64, 64), (64, 128), (80, 128), (96, 128), (112, 128), (128, 128),   # tcgen05 kernel
          (128, 160), (128, 192), (128, 224),                                     # tcgen05 wide kernel
          (16, 32), (32, 128), (128, 32), (16, 256), (256, 16), (128, 112),       # mma.sync kernel
          (224, 64), (64, 224),
          (8, 8), (6, 10), (16, 48), (32, 32), (2, 3 * 2)]                        # CUDA-core kernel


@pytest.fixture(params=[0, 1, 2], ids=["tq_default", "tq_mma_sync", "tq_simt"])
def tq_impl(request):
    fq.fq_set_tq_impl(request.param)
    yield request.param
    fq.fq_set_tq_impl(0)


@pytest.mark.parametrize("n1,n2", SHAPES)
@pytest.mark.parametrize("alpha", [1.0, 0.9])
@pytest.mark.parametrize("tdtype", [torch.float16, torch.bfloat16])
def test_transform_quant_vs_oracle(n1, n2, alpha, tdtype, tq_impl):
    if tq_impl == 2 and n1 * n2 > 16384:
        pytest.skip("CUDA-core kernel: smem bound")
    T = 300 if n1 * n2 <= 16384 else 137                  # several tiles/CTAs and a ragged tail
    x, p1, p2 = make_inputs(T, n1, n2, seed=n1 + n2, tdtype=tdtype)
    q, s, y = run_tq(x, p1, p2, alpha, n1, n2)
    qo, so, yo = O.transform_quant(x.float().numpy(), p1.float().numpy(), p2.float().numpy(), alpha)
    st = parity.check_transform(q, s, y, yo, qo, so, label=f"{n1}x{n2} a={alpha} {tdtype}")
    assert st["mismatch_frac"] <= parity.MISMATCH_FRAC


@pytest.mark.parametrize("n1,n2", [(16, 32), (64, 64), (112, 128)])
def test_transform_special_matrices(n1, n2):
    """Identity P: y = x exactly, so codes are the oracle's on the raw activations; Hadamard:
    a spike spreads to +-7 everywhere; permutation: codes are permuted identity codes."""
    T = 64
    x, _, _ = make_inputs(T, n1, n2, seed=3)
    eye1, eye2 = torch.eye(n1, dtype=torch.float16), torch.eye(n2, dtype=torch.float16)
    q, s, y = run_tq(x, eye1, eye2, 1.0, n1, n2)
    assert np.array_equal(y, x.float().numpy())
    qo, so, yo = O.transform_quant(x.float().numpy(), eye1.float().numpy(), eye2.float().numpy(), 1.0)
    parity.check_transform(q, s, y, yo, qo, so, tau=1e-4, label="identity")
    if (n1 & (n1 - 1)) == 0 and (n2 & (n2 - 1)) == 0:
        h1 = torch.from_numpy(synth.hadamard(n1, np.float32)).half()
        h2 = torch.from_numpy(synth.hadamard(n2, np.float32)).half()
        spike = torch.zeros((4, n1 * n2), dtype=torch.float16)
        spike[0, 3] = 2.0
        spike[1, n1 * n2 - 1] = -300.0
        spike[2, 7] = 0.001
        q, s, y = run_tq(spike, h1, h2, 1.0, n1, n2)
        codes = O.unpack_int4(q)
        assert np.all(np.abs(codes[:3]) == 7)
        assert np.all(codes[3] == 0) and s[3] == 1.0      # all-zero token: s = 1, codes 0
    p1 = torch.from_numpy(synth.permutation(n1, seed=1, dtype=np.float32)).half()
    p2 = torch.from_numpy(synth.permutation(n2, seed=2, dtype=np.float32)).half()
    q, s, y = run_tq(x, p1, p2, 1.0, n1, n2)
    perm = np.kron(p1.float().numpy(), p2.float().numpy()).argmax(axis=0)
    assert np.array_equal(y, x.float().numpy()[:, perm])


@pytest.mark.parametrize("n1,n2", [(64, 64), (64, 128), (112, 128), (128, 224)])
@pytest.mark.parametrize("T", [1, 2, 3, 5, 149, 295, 297, 1031])
def test_transform_tile_tails(n1, n2, T):
    """Token counts around the tile size (2 tokens for n1 = 64) and the grid size (148 SMs):
    the TMA zero-fills tokens past T and the kernel must not write them."""
    x, p1, p2 = make_inputs(T, n1, n2, seed=T)
    q = torch.full((T + 2, n1 * n2 // 2), 0xAB, dtype=torch.uint8, device=DEV)
    s = torch.full((T + 2,), -1.0, dtype=torch.float32, device=DEV)
    fq.fq_transform_quant(x.to(DEV), n1, n2, p1.to(DEV), p2.to(DEV), 0.9, q[:T], s[:T])
    torch.cuda.synchronize()
    assert np.all(np_of(q[T:]) == 0xAB) and np.all(np_of(s[T:]) == -1.0)     # nothing past T
    qo, so, yo = O.transform_quant(x.float().numpy(), p1.float().numpy(), p2.float().numpy(), 0.9)
    parity.check_transform(np_of(q[:T]), np_of(s[:T]), None, yo, qo, so, label=f"tail T={T}")


@pytest.mark.parametrize("alpha", [1.0, 0.9])
@pytest.mark.parametrize("tdtype", [torch.float16, torch.bfloat16])
def test_transform_wide_n2_256(alpha, tdtype):
    """n1 x n2 = 128 x 256 exists only on the wide tcgen05 kernel (P2 alone is 128 KB of smem)."""
    x, p1, p2 = make_inputs(300, 128, 256, seed=31, tdtype=tdtype)
    q, s, y = run_tq(x, p1, p2, alpha, 128, 256)
    qo, so, yo = O.transform_quant(x.float().numpy(), p1.float().numpy(), p2.float().numpy(), alpha)
    parity.check_transform(q, s, y, yo, qo, so, label="128x256")


@pytest.mark.parametrize("n1", [32, 64])
@pytest.mark.parametrize("alpha", [1.0, 0.9])
@pytest.mark.parametrize("tdtype", [torch.float16, torch.bfloat16])
def test_transform_p2_identity(n1, alpha, tdtype):
    """p2 = NULL: the paper's online o_proj transform P_o (a x a) (x) I_{d_head} (PAPER.md:297,
    726), a = n1 heads of 128; the oracle applies the explicit identity."""
    n2, T = 128, 301
    x, p1, _ = make_inputs(T, n1, n2, seed=n1 + 7, tdtype=tdtype)
    q, s, y = fq.transform_f32(x.to(DEV), n1, n2, p1.to(DEV), None, alpha)
    torch.cuda.synchronize()
    qo, so, yo = O.transform_quant(x.float().numpy(), p1.float().numpy(), np.eye(n2), alpha)
    st = parity.check_transform(np_of(q), np_of(s), np_of(y), yo, qo, so, label=f"P_o x I a={n1}")
    assert st["mismatch_frac"] <= parity.MISMATCH_FRAC
    q2, s2 = fq.transform_quant(x.to(DEV), n1, n2, p1.to(DEV), None, alpha)
    torch.cuda.synchronize()
    assert torch.equal(q2.cpu(), q.cpu()) and torch.equal(s2.cpu(), s.cpu())


@pytest.mark.parametrize("n1", [32, 64])
@pytest.mark.parametrize("impl", [0, 1], ids=["tcgen05", "mma_sync"])
@pytest.mark.parametrize("T", [1, 2, 3, 149, 297])
def test_transform_p2_identity_kernels_and_tails(n1, impl, T):
    """P2 = I on both kernels (tcgen05 stage-1-only, the default; legacy mma.sync) at token counts
    around the tile (1 or 2 tokens) and grid sizes: nothing written past T, parity with the oracle."""
    n2 = 128
    x, p1, _ = make_inputs(T, n1, n2, seed=T + n1)
    q = torch.full((T + 2, n1 * n2 // 2), 0xAB, dtype=torch.uint8, device=DEV)
    s = torch.full((T + 2,), -1.0, dtype=torch.float32, device=DEV)
    fq.fq_set_tq_impl(impl)
    try:
        fq.fq_transform_quant(x.to(DEV), n1, n2, p1.to(DEV), None, 0.9, q[:T], s[:T])
        torch.cuda.synchronize()
    finally:
        fq.fq_set_tq_impl(0)
    assert np.all(np_of(q[T:]) == 0xAB) and np.all(np_of(s[T:]) == -1.0)
    qo, so, yo = O.transform_quant(x.float().numpy(), p1.float().numpy(), np.eye(n2), 0.9)
    parity.check_transform(np_of(q[:T]), np_of(s[:T]), None, yo, qo, so, label=f"P2=I impl {impl} T={T}")


@pytest.mark.parametrize("n1", [32, 64])
@pytest.mark.parametrize("alpha", [1.0, 0.9])
@pytest.mark.parametrize("tdtype", [torch.float16, torch.bfloat16])
def test_transform_p2_identity_asym(n1, alpha, tdtype):
    """FQ_ASYM with P2 = I (tcgen05 kernel): codes, scales and zero points against the oracle's
    asymmetric quantizer of P1^T V (reading R19, R22)."""
    n2, T = 128, 211
    x, p1, _ = make_inputs(T, n1, n2, seed=n1 + 11, tdtype=tdtype)
    q, s, z = fq.transform_quant_asym(x.to(DEV), n1, n2, p1.to(DEV), None, alpha)
    torch.cuda.synchronize()
    qo, so, zo, yo = O.transform_quant_asym(x.float().numpy(), p1.float().numpy(), np.eye(n2), alpha)
    parity.check_asym(np_of(q), np_of(s), np_of(z), yo, alpha, qo, so, zo, label=f"asym P2=I a={n1}")


def test_gpu_weight_prep_p2_identity():
    """fq_prepare_weight with p2 = NULL: W' = P1^{-1} W~ (P2 = I, so P2^{-T} = I); parity as in
    test_gpu_weight_prep_matches_oracle (oracle with the fp16-rounded P1^{-T} and the identity)."""
    n1, n2, N = 32, 128, 264
    w = torch.from_numpy(synth.weights(N, n1 * n2, seed=3, dtype=np.float32)).half()
    p1 = torch.from_numpy(synth.well_conditioned(n1, seed=3, tag="p1", dtype=np.float32)).half()
    qw, sw = fq.prepare_weight(w.to(DEV), n1, n2, p1.to(DEV), None, 1.0)
    torch.cuda.synchronize()
    wf, p1f = w.float().numpy().astype(np.float64), p1.float().numpy().astype(np.float64)
    p1i_t = torch.from_numpy(np.linalg.inv(p1f).T.copy()).half().float().numpy()
    qo, so, yo = O.transform_quant(wf, p1i_t, np.eye(n2), 1.0)
    parity.check_transform(np_of(qw), np_of(sw), None, yo, qo, so, label="weight prep P2 = I")


def test_transform_overflow_stress_fp16():
    """A token at +-60000 in every channel: the fp16 intermediate must not overflow (exact
    power-of-two prescale), and zero / tiny tokens must not underflow."""
    n1, n2, T = 64, 64, 8
    g = np.random.default_rng(0)
    x = np.where(g.random((T, n1 * n2)) < 0.5, -60000.0, 60000.0).astype(np.float16)
    x[1] = 0
    x[2] = (g.standard_normal(n1 * n2) * 1e-4).astype(np.float16)
    p1 = synth.well_conditioned(n1, seed=5, tag="p1")
    p2 = synth.well_conditioned(n2, seed=5, tag="p2")
    q, s, y = run_tq(torch.from_numpy(x), torch.from_numpy(p1), torch.from_numpy(p2), 1.0, n1, n2)
    assert np.all(np.isfinite(y)) and np.all(np.isfinite(s))
    qo, so, yo = O.transform_quant(x, p1, p2, 1.0)
    parity.check_transform(q, s, y, yo, qo, so, label="overflow stress")


def test_transform_strided_rows_and_empty():
    n1, n2, T = 64, 64, 33
    x, p1, p2 = make_inputs(T, n1, n2, seed=4)
    xb = torch.zeros((T, n1 * n2 + 64), dtype=torch.float16)
    xb[:, : n1 * n2] = x
    xd = xb.to(DEV)[:, : n1 * n2]                       # ldx = n + 64
    q, s = fq.transform_quant(xd, n1, n2, p1.to(DEV), p2.to(DEV), 0.95)
    qo, so, yo = O.transform_quant(x.float().numpy(), p1.float().numpy(), p2.float().numpy(), 0.95)
    parity.check_transform(np_of(q), np_of(s), None, yo, qo, so, label="strided")
    q0, s0 = fq.transform_quant(xd[:0], n1, n2, p1.to(DEV), p2.to(DEV), 1.0)
    assert q0.shape == (0, n1 * n2 // 2)


# GEMM implementations (fq_set_gemm_impl): 0 pair kernel, tile width per shape; 1 legacy mma.sync;
# 2 single-CTA tcgen05; 3 / 4 / 5 / 7 pair kernel with the tile width forced to 192 / 160 / 128 / 256.
GEMM_IMPLS = [0, 1, 2, 3, 4, 5, 7]


@pytest.mark.parametrize("impl", GEMM_IMPLS)
@pytest.mark.parametrize("T,N,K", [(1, 8, 32), (37, 24, 96), (128, 256, 128), (300, 520, 4096),
                                   (2048, 4096, 4096), (257, 4096, 14336), (64, 28672, 4096), (513, 200, 352),
                                   (700, 168, 4096)])
def test_gemm_i32_bit_exact(impl, T, N, K):
    qa = synth.random_codes(T, K, seed=T, tag="qa")
    qw = synth.random_codes(N, K, seed=N, tag="qw")
    fq.fq_set_gemm_impl(impl)
    try:
        acc = fq.w4a4_gemm_i32(to_dev(O.pack_int4(qa)), to_dev(O.pack_int4(qw)))
        torch.cuda.synchronize()
    finally:
        fq.fq_set_gemm_impl(0)
    ref = O.int_gemm(qa, qw)
    assert np.array_equal(np_of(acc).astype(np.int64), ref)


# Decode kernel (impl 6; the default for T <= 64): swapped operands, K split across a cluster of
# S CTAs reduced through distributed shared memory.  The shapes cover S = 1 (one K-block;
# 224 feature blocks), S = 4 (ragged N and K), S = 6 (qkv) and S = 8 (down_proj), ragged token
# counts (MMA N = T rounded up to 16) and the 64-token maximum.
DEC_SHAPES = [(8, 32), (24, 96), (264, 416), (200, 352), (6144, 4096), (4096, 14336), (28672, 4096)]


@pytest.mark.parametrize("impl", [0, 6])
@pytest.mark.parametrize("T", [1, 7, 16, 33, 64])
@pytest.mark.parametrize("N,K", DEC_SHAPES)
def test_gemm_decode_i32_bit_exact(impl, T, N, K):
    qa = synth.random_codes(T, K, seed=T + 11, tag="qa")
    qw = synth.random_codes(N, K, seed=N + 11, tag="qw")
    fq.fq_set_gemm_impl(impl)
    try:
        acc = fq.w4a4_gemm_i32(to_dev(O.pack_int4(qa)), to_dev(O.pack_int4(qw)))
        torch.cuda.synchronize()
    finally:
        fq.fq_set_gemm_impl(0)
    assert np.array_equal(np_of(acc).astype(np.int64), O.int_gemm(qa, qw))


def test_gemm_decode_extreme_values_and_limits():
    """Extreme codes at the largest K of the configs (|acc| = 64 K) through an 8-way split, and
    T = 65 (one past the decode kernel's limit) is refused when the decode kernel is forced."""
    T, N, K = 64, 264, 28672
    qa = np.full((T, K), -8, np.int8)
    qw = np.full((N, K), -8, np.int8)
    qw[1::2] = 7
    fq.fq_set_gemm_impl(6)
    try:
        acc = fq.w4a4_gemm_i32(to_dev(O.pack_int4(qa)), to_dev(O.pack_int4(qw)))
        torch.cuda.synchronize()
        assert np.array_equal(np_of(acc).astype(np.int64), O.int_gemm(qa, qw))
        qa65 = to_dev(O.pack_int4(np.zeros((65, 64), np.int8)))
        qw65 = to_dev(O.pack_int4(np.zeros((8, 64), np.int8)))
        with pytest.raises(RuntimeError, match="ENOTSUP"):
            fq.w4a4_gemm_i32(qa65, qw65)
    finally:
        fq.fq_set_gemm_impl(0)


@pytest.mark.parametrize("out_dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("T", [1, 29, 64])
def test_w4a4_linear_dequant_decode(out_dtype, T):
    N, K = 776, 2080
    qa = synth.random_codes(T, K, seed=3, tag="qa")
    qw = synth.random_codes(N, K, seed=4, tag="qw")
    sa = synth.random_scales(T, seed=3, tag="sa")
    sw = synth.random_scales(N, seed=4, tag="sw")
    y = fq.w4a4_linear(to_dev(O.pack_int4(qa)), to_dev(sa), to_dev(O.pack_int4(qw)), to_dev(sw), out_dtype)
    torch.cuda.synchronize()
    ref = O.w4a4_linear(qa, sa, qw, sw)
    parity.check_output(np_of(y), ref, label="w4a4_linear decode")
    ulp = 2.0 ** -10 if out_dtype == torch.float16 else 2.0 ** -7
    assert np.all(np.abs(np_of(y) - ref) <= ulp * np.abs(ref) + 1e-6)


def test_gemm_i32_extreme_values():
    T, N, K = 130, 264, 28672
    qa = np.full((T, K), -8, np.int8)
    qw = np.full((N, K), -8, np.int8)
    qw[1::2] = 7
    acc = fq.w4a4_gemm_i32(to_dev(O.pack_int4(qa)), to_dev(O.pack_int4(qw)))
    ref = O.int_gemm(qa, qw)
    assert np.array_equal(np_of(acc).astype(np.int64), ref)


@pytest.mark.parametrize("out_dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("impl", GEMM_IMPLS)
def test_w4a4_linear_dequant(out_dtype, impl):
    T, N, K = 333, 776, 2048
    qa = synth.random_codes(T, K, seed=1, tag="qa")
    qw = synth.random_codes(N, K, seed=2, tag="qw")
    sa = synth.random_scales(T, seed=1, tag="sa")
    sw = synth.random_scales(N, seed=2, tag="sw")
    fq.fq_set_gemm_impl(impl)
    try:
        y = fq.w4a4_linear(to_dev(O.pack_int4(qa)), to_dev(sa), to_dev(O.pack_int4(qw)), to_dev(sw), out_dtype)
        torch.cuda.synchronize()
    finally:
        fq.fq_set_gemm_impl(0)
    ref = O.w4a4_linear(qa, sa, qw, sw)
    parity.check_output(np_of(y), ref, label="w4a4_linear")
    # fp16/bf16 rounding of an fp32 product: element-wise within a few ulps of the reference
    ulp = 2.0 ** -10 if out_dtype == torch.float16 else 2.0 ** -7
    assert np.all(np.abs(np_of(y) - ref) <= ulp * np.abs(ref) + 1e-6)


def _chain(cfg, lin, tokens, seed=0, alpha=0.9, full_weight_prep=True):
    T = cfg["T"]
    n1, n2, N, K = lin.n1, lin.n2, lin.N, lin.K
    x = synth.activations(T, K, seed=seed, tag=lin.name)
    p1 = synth.well_conditioned(n1, seed=seed, tag=lin.name + "/p1")
    p2 = synth.well_conditioned(n2, seed=seed, tag=lin.name + "/p2")
    if full_weight_prep:
        w = synth.weights(N, K, seed=seed, tag=lin.name)
        qw, sw, _ = O.prepare_weight(w, p1, p2, 1.0)
    else:   # large configs: synthetic pre-quantized weights (the GEMM is weight-agnostic)
        qw = synth.random_codes(N, K, seed=seed, tag=lin.name + "/qw")
        sw = synth.random_scales(N, seed=seed, tag=lin.name + "/sw")
    sw32 = np.asarray(sw, np.float32)
    xd = to_dev(x)
    qa, sa = fq.transform_quant(xd, n1, n2, to_dev(p1), to_dev(p2), alpha)
    y = fq.w4a4_linear(qa, sa, to_dev(O.pack_int4(qw)), to_dev(sw32))
    yfull = fq.flatquant_linear(xd, n1, n2, to_dev(p1), to_dev(p2), alpha, to_dev(O.pack_int4(qw)), to_dev(sw32))
    torch.cuda.synchronize()
    assert torch.equal(y, yfull)                        # the fused entry point is the same path
    rows = tokens if tokens is not None else np.arange(T)
    rows = np.asarray(rows)
    qo, so, yo = O.transform_quant(x[rows], p1, p2, alpha)
    parity.check_transform(np_of(qa[torch.as_tensor(rows, device=DEV)]), np_of(sa)[rows], None, yo, qo, so,
                           label=f"{lin.name} transform")
    out_o = O.w4a4_linear(qo, so, qw, sw32.astype(np.float64))
    qa_rows = O.unpack_int4(np_of(qa[torch.as_tensor(rows, device=DEV)]))
    out_same = O.w4a4_linear(qa_rows, np_of(sa)[rows].astype(np.float64), qw, sw32.astype(np.float64))
    return parity.check_output(np_of(y)[rows], out_o, out_same, label=f"{lin.name} output")


def sample_rows(T, seed=0):
    if T <= 512:
        return None
    g = np.random.default_rng(seed)
    return np.unique(np.concatenate([np.arange(256), g.choice(np.arange(256, T), 256, replace=False)]))


@pytest.mark.parametrize("cfg_name", ["C1", "C2"])
def test_chain_full(cfg_name):
    cfg = synth.config(cfg_name)
    for lin in cfg["linears"]:
        _chain(cfg, lin, None)


@pytest.mark.parametrize("cfg_name", ["C3", "C4"])
def test_chain_llama3_8b(cfg_name):
    cfg = synth.config(cfg_name)
    for lin in cfg["linears"]:
        _chain(cfg, lin, sample_rows(cfg["T"]), full_weight_prep=(lin.N * lin.K <= 4096 * 14336))


def test_chain_llama3_70b_sampled():
    cfg = synth.config("C5")
    for lin in cfg["linears"]:
        _chain(cfg, lin, sample_rows(cfg["T"]), full_weight_prep=False)


def test_determinism():
    cfg = synth.config("C2")
    lin = cfg["linears"][0]
    x, p1, p2 = make_inputs(cfg["T"], lin.n1, lin.n2, seed=9)
    qw = to_dev(O.pack_int4(synth.random_codes(lin.N, lin.K, seed=9)))
    sw = to_dev(synth.random_scales(lin.N, seed=9))
    outs = [fq.flatquant_linear(x.to(DEV), lin.n1, lin.n2, p1.to(DEV), p2.to(DEV), 0.9, qw, sw) for _ in range(2)]
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("n1,n2,N,tdtype,alpha_w", [(64, 64, 512, torch.float16, 1.0),
                                                    (64, 128, 264, torch.bfloat16, 0.95),
                                                    (112, 128, 136, torch.float16, 1.0),
                                                    (16, 32, 72, torch.float16, 0.9)])
def test_gpu_weight_prep_matches_oracle(n1, n2, N, tdtype, alpha_w):
    """NEXT-2: fq_prepare_weight computes W' = P1^{-1} W~ P2^{-T} on the GPU:
    float64 Gauss-Jordan inverses rounded to the weights' dtype, then the activation kernel with
    (P1^{-T}, P2^{-T}, alpha_w).  Parity: the oracle's transform+quant of W with the inverses
    numpy computes in float64 and rounds to the same dtype (bars 2-3 per output channel); the
    dequantized weights against the exact float64 W' within the 4-bit RTN step; colsum_w exact."""
    w = torch.from_numpy(synth.weights(N, n1 * n2, seed=3, dtype=np.float32)).to(tdtype)
    p1 = torch.from_numpy(synth.well_conditioned(n1, seed=3, tag="p1", dtype=np.float32)).to(tdtype)
    p2 = torch.from_numpy(synth.well_conditioned(n2, seed=3, tag="p2", dtype=np.float32)).to(tdtype)
    qw, sw, cs = fq.prepare_weight(w.to(DEV), n1, n2, p1.to(DEV), p2.to(DEV), alpha_w, with_colsum=True)
    torch.cuda.synchronize()
    wf, p1f, p2f = (t.float().numpy().astype(np.float64) for t in (w, p1, p2))
    p1i_t = torch.from_numpy(np.linalg.inv(p1f).T.copy()).to(tdtype).float().numpy()
    p2i_t = torch.from_numpy(np.linalg.inv(p2f).T.copy()).to(tdtype).float().numpy()
    qo, so, yo = O.transform_quant(wf, p1i_t, p2i_t, alpha_w)
    parity.check_transform(np_of(qw), np_of(sw), None, yo, qo, so, label=f"weight prep {n1}x{n2}")
    codes = O.unpack_int4(np_of(qw))
    assert np.array_equal(np_of(cs).astype(np.int64), codes.astype(np.int64).sum(1))
    _, _, wp = O.prepare_weight(wf, p1f, p2f, alpha_w)
    deq = O.dequantize_rows(codes, np_of(sw).astype(np.float64))
    step = np_of(sw).astype(np.float64)[:, None]
    inside = np.abs(wp) <= 7 * step
    tol = 0.5 * step + 2e-2 * np.abs(wp).max(1, keepdims=True)
    assert np.all((np.abs(deq - wp) <= tol)[inside])


def test_gpu_weight_prep_singular():
    """A singular P (a zero row) or one whose inverse overflows fp16 (1e-5 I) is reported as
    FQ_ESINGULAR before anything is quantized."""
    n1, n2, N = 16, 32, 8
    w = to_dev(synth.weights(N, n1 * n2, seed=1))
    p2 = to_dev(synth.well_conditioned(n2, seed=1, tag="p2"))
    bad = synth.well_conditioned(n1, seed=1, tag="p1").copy()
    bad[3] = 0
    for p1 in (to_dev(bad), to_dev((np.eye(n1) * 1e-5).astype(np.float16))):
        with pytest.raises(fq.FlatQuantError) as e:
            fq.prepare_weight(w, n1, n2, p1, p2, 1.0)
        assert e.value.status == fq.FQ_ESINGULAR


# ---------------------------------------------------------------- asymmetric mode (NEXT-1, R19)
@pytest.mark.parametrize("n1,n2", [(64, 64), (64, 128), (112, 128), (128, 224), (16, 32), (8, 8)])
@pytest.mark.parametrize("alpha", [1.0, 0.9])
@pytest.mark.parametrize("tdtype", [torch.float16, torch.bfloat16])
def test_transform_quant_asym_vs_oracle(n1, n2, alpha, tdtype):
    """FQ_ASYM: codes q in [0, 15] (stored q - 8), zero points z (stored z - 8) and scales against
    the oracle.  Compared on the grid index q - z (a +-1 zero-point flip at a near-tie of
    -lo/s shifts every code of its token but not q - z); mismatches only at near-ties of y/s or
    at the clamp, by +-1, in <= 0.1% of the elements."""
    T = 203
    x, p1, p2 = make_inputs(T, n1, n2, seed=n1 * 3 + n2, tdtype=tdtype)
    q, s, z = fq.transform_quant_asym(x.to(DEV), n1, n2, p1.to(DEV), p2.to(DEV), alpha)
    torch.cuda.synchronize()
    qo, so, zo, yo = O.transform_quant_asym(x.float().numpy(), p1.float().numpy(), p2.float().numpy(), alpha)
    parity.check_asym(np_of(q), np_of(s), np_of(z), yo, alpha, qo, so, zo, label=f"asym {n1}x{n2}")


def test_weight_colsum_exact():
    qw = synth.random_codes(777, 4096, seed=5)
    cs = fq.weight_colsum(to_dev(O.pack_int4(qw)))
    torch.cuda.synchronize()
    assert np.array_equal(np_of(cs).astype(np.int64), qw.astype(np.int64).sum(1))


@pytest.mark.parametrize("impl,T", [(0, 1037), (4, 1037), (7, 1037), (0, 64), (6, 23)])
@pytest.mark.parametrize("out_dtype", [torch.float16, torch.bfloat16])
def test_asym_linear_vs_oracle(out_dtype, impl, T):
    """Asymmetric activations through the GEMM: Y = s_a s_w (acc - (z - 8) colsum_w) equals the
    oracle's dequantized product of the GPU's own codes (per token, fp16/bf16 output rounding),
    and the whole chain stays within the end-to-end Frobenius bar of the oracle's codes."""
    n1, n2, N = 64, 64, 1544
    x, p1, p2 = make_inputs(T, n1, n2, seed=17)
    w = synth.weights(N, n1 * n2, seed=17)
    qw, sw, _ = O.prepare_weight(w, p1.float().numpy(), p2.float().numpy(), 1.0)
    sw32 = sw.astype(np.float32)
    qw_d = to_dev(O.pack_int4(qw))
    q, s, z = fq.transform_quant_asym(x.to(DEV), n1, n2, p1.to(DEV), p2.to(DEV), 0.9)
    cs = fq.weight_colsum(qw_d)
    fq.fq_set_gemm_impl(impl)
    try:
        y = fq.w4a4_linear(q, s, qw_d, to_dev(sw32), out_dtype, za=z, colsum_w=cs)
        torch.cuda.synchronize()
    finally:
        fq.fq_set_gemm_impl(0)
    qg = O.unpack_int4(np_of(q)).astype(np.int64) + 8
    zg = np_of(z).astype(np.int64) + 8
    same = O.w4a4_linear_asym(qg, np_of(s).astype(np.float64), zg, qw, sw32.astype(np.float64))
    ulp = 2.0 ** -10 if out_dtype == torch.float16 else 2.0 ** -7
    assert np.all(np.abs(np_of(y) - same) <= ulp * np.abs(same) + 1e-6)
    qo, so, zo, _ = O.transform_quant_asym(x.float().numpy(), p1.float().numpy(), p2.float().numpy(), 0.9)
    ref = O.w4a4_linear_asym(qo, so, zo, qw, sw32.astype(np.float64))
    parity.check_output(np_of(y), ref, same, label="asym linear")


def test_host_buffer_entry_points_match_device_path():
    """fq_flatquant_linear_host (synchronous) and fq_flatquant_linear_host_async (two streams,
    caller synchronises) give bit-identical outputs to the device-buffer entry point."""
    T, n1, n2, N = 300, 64, 64, 520
    x, p1, p2 = make_inputs(T, n1, n2, seed=41)
    qw = synth.random_codes(N, n1 * n2, seed=41, tag="qw")
    sw = to_dev(synth.random_scales(N, seed=41, tag="sw"))
    qwd, p1d, p2d = to_dev(O.pack_int4(qw)), p1.to(DEV), p2.to(DEV)
    ref = fq.flatquant_linear(x.to(DEV), n1, n2, p1d, p2d, 0.9, qwd, sw)
    torch.cuda.synchronize()
    xh = x.contiguous().pin_memory()
    outs = []
    for sync, stream in ((True, None), (False, torch.cuda.Stream()), (False, torch.cuda.Stream())):
        yh = torch.empty((T, N), dtype=torch.float16).pin_memory()
        xd, yd = torch.empty_like(x, device=DEV), torch.empty((T, N), dtype=torch.float16, device=DEV)
        qws = torch.empty((T, n1 * n2 // 2), dtype=torch.uint8, device=DEV)
        sws = torch.empty((T,), dtype=torch.float32, device=DEV)
        fq.fq_flatquant_linear_host(xh, xd, n1, n2, p1d, p2d, 0.9, qwd, sw, yh, yd, qws, sws, stream=stream, sync=sync)
        outs.append((yh, stream, (xd, yd, qws, sws)))
    torch.cuda.synchronize()
    for yh, _, _ in outs:
        assert torch.equal(yh, ref.cpu())
