"""GPU checks of the ABI's edges (round-2 review items): the K range of the widened int32
accumulator, bf16 transforms outside fp16 range, the programmatic-dependent-launch parameter
hazard, and the Python binding's shape checks.  Expected values are closed forms or the oracle.
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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def packed_const_rows(vals, K):
    """[len(vals), K/2] packed codes whose row r holds the code vals[r] in every column."""
    codes = np.repeat(np.asarray(vals, np.int8)[:, None], K, axis=1)
    return O.pack_int4(codes)


# ------------------------------------------------------------------ K range (flatquant.h)
@pytest.mark.parametrize("impl,T", [(0, 130), (2, 130), (6, 64), (1, 37)])
def test_gemm_k_cap_symmetric_bit_exact(impl, T):
    """K = 131040 (largest K % 32 == 0 below the cap): all -8 activations against -8 / 7 weights
    give |acc| = 64 K, so the widened accumulator holds 256 * 64 * 131040 = 2^31 - 2^19 without
    wrapping.  Closed form acc[t, o] = a_t b_o K."""
    K, N = 131040, 264
    a = np.full(T, -8, np.int8)
    a[1::3] = 7
    b = np.where(np.arange(N) % 2 == 0, -8, 7).astype(np.int8)
    fq.fq_set_gemm_impl(impl)
    try:
        acc = fq.w4a4_gemm_i32(dev(packed_const_rows(a, K)), dev(packed_const_rows(b, K)))
        torch.cuda.synchronize()
    finally:
        fq.fq_set_gemm_impl(0)
    ref = a.astype(np.int64)[:, None] * b.astype(np.int64)[None, :] * K
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), ref)


@pytest.mark.parametrize("K", [65504, 131040])
@pytest.mark.parametrize("impl,T", [(0, 130), (6, 40)])
def test_gemm_k_cap_asymmetric_exact(K, impl, T):
    """Asymmetric activations at the caps: stored codes q - 8 = -8 with z - 8 = 7 (q - z = -15)
    against weights -8 give acc_true = 120 K (= 15.7 M at K = 131040).  Formed in the x256 domain
    this wrapped int32 from K = 65536; the epilogue now corrects after the exact >> 8.  With
    s_a = 2^-24 and s_w = 1 the fp16 output is the fp16 rounding of 120 K 2^-24."""
    N = 264
    qa = dev(packed_const_rows(np.full(T, -8), K))
    za = torch.full((T,), 7, dtype=torch.int8, device=DEV)
    qw = dev(packed_const_rows(np.full(N, -8), K))
    cs = fq.weight_colsum(qw)
    sa = torch.full((T,), 2.0 ** -24, dtype=torch.float32, device=DEV)
    sw = torch.ones((N,), dtype=torch.float32, device=DEV)
    fq.fq_set_gemm_impl(impl)
    try:
        y = fq.w4a4_linear(qa, sa, qw, sw, torch.float16, za=za, colsum_w=cs)
        torch.cuda.synchronize()
    finally:
        fq.fq_set_gemm_impl(0)
    assert np.all(cs.cpu().numpy() == -8 * K)
    expect = np.float16(120.0 * K * 2.0 ** -24)
    assert np.all(y.cpu().numpy() == expect)


def test_gemm_k_cap_rejected_through_binding():
    qa = torch.zeros((8, 131072 // 2), dtype=torch.uint8, device=DEV)
    qw = torch.zeros((16, 131072 // 2), dtype=torch.uint8, device=DEV)
    with pytest.raises(RuntimeError, match="ENOTSUP"):
        fq.w4a4_gemm_i32(qa, qw)


# ------------------------------------------------------------------ bf16 P outside fp16 range
@pytest.mark.parametrize("tq_impl,n1,n2", [(0, 64, 64), (0, 112, 128), (0, 128, 224), (1, 64, 64), (1, 128, 112),
                                           (2, 16, 32)])
@pytest.mark.parametrize("p2_scale", [1e5, 2.0 ** 20, 2.0 ** -30])
def test_bf16_p2_beyond_fp16_range(tq_impl, n1, n2, p2_scale):
    """The second Kronecker stage runs in fp16 (reading R9); a bf16 P2 whose entries leave fp16
    range (1e5, 2^20) or sit in its subnormals (2^-30) must still match the oracle: the kernels
    scale P2 by a power of two into range and divide it out of the result exactly.  P1 carries
    the inverse scale, so y keeps the magnitude of x.  Also P1 = 1e-5 I, P2 = 1e5 I."""
    T = 150
    x = torch.from_numpy(synth.activations(T, n1 * n2, seed=5, dtype=np.float32)).to(torch.bfloat16)
    p1 = torch.from_numpy(synth.well_conditioned(n1, seed=5, tag="p1", dtype=np.float32) / p2_scale).to(torch.bfloat16)
    p2 = torch.from_numpy(synth.well_conditioned(n2, seed=5, tag="p2", dtype=np.float32) * p2_scale).to(torch.bfloat16)
    cases = [(p1, p2)]
    if p2_scale == 1e5:
        cases.append(((torch.eye(n1) * 1e-5).to(torch.bfloat16), (torch.eye(n2) * 1e5).to(torch.bfloat16)))
    fq.fq_set_tq_impl(tq_impl)
    try:
        for a1, a2 in cases:
            q, s, y = fq.transform_f32(x.to(DEV), n1, n2, a1.to(DEV), a2.to(DEV), 0.9)
            torch.cuda.synchronize()
            assert torch.isfinite(y).all() and torch.isfinite(s).all()
            qo, so, yo = O.transform_quant(x.float().numpy(), a1.float().numpy(), a2.float().numpy(), 0.9)
            parity.check_transform(q.cpu().numpy(), s.cpu().numpy(), y.cpu().numpy(), yo, qo, so,
                                   label=f"bf16 P2 x{p2_scale} {n1}x{n2} impl {tq_impl}")
    finally:
        fq.fq_set_tq_impl(0)


# ------------------------------------------------------------------ PDL parameter hazard
def test_pdl_parameter_written_by_preceding_kernel():
    """A kernel's parameters may be the outputs of the kernel right before it on the stream:
    (i) fq_transform_quant writes packed codes + scales that the next fq_w4a4_linear takes as
    its WEIGHTS (qw, sw) -- decode and prefill GEMMs; (ii) a GEMM's fp16 output [64, 64] is the
    P1 of the next transform.  The library detects the overlap and reads such parameters after
    griddepcontrol.wait; results equal a run with a full synchronisation between the calls."""
    torch.manual_seed(0)
    n1 = n2 = 64
    K = n1 * n2
    Nw = 6144                                        # a long weight-producing transform
    wsrc = torch.from_numpy(synth.weights(Nw, K, seed=9)).to(DEV)
    e1 = torch.eye(n1, dtype=torch.float16, device=DEV)
    e2 = torch.eye(n2, dtype=torch.float16, device=DEV)
    qa, sa = fq.transform_quant(torch.from_numpy(synth.activations(300, K, seed=9)).to(DEV), n1, n2, e1, e2, 0.9)
    torch.cuda.synchronize()
    for T in (48, 300):                              # decode kernel (weights before the wait) and pair kernel
        outs = []
        for sync in (True, False):
            qw = torch.full((Nw, K // 2), 0x77, dtype=torch.uint8, device=DEV)
            sw = torch.full((Nw,), float("nan"), dtype=torch.float32, device=DEV)
            torch.cuda.synchronize()
            fq.fq_transform_quant(wsrc, n1, n2, e1, e2, 1.0, qw, sw)
            if sync:
                torch.cuda.synchronize()
            y = fq.w4a4_linear(qa[:T], sa[:T], qw, sw)
            torch.cuda.synchronize()
            outs.append(y)
        assert torch.isfinite(outs[0]).all()
        assert torch.equal(outs[0], outs[1])
    # (ii) GEMM output -> next transform's P1
    qa64, sa64 = qa[:64], sa[:64]
    qwp, swp = fq.transform_quant(torch.from_numpy(synth.weights(64, K, seed=10)).to(DEV), n1, n2, e1, e2, 1.0)
    x = torch.from_numpy(synth.activations(1000, K, seed=11)).to(DEV)
    res = []
    for sync in (True, False):
        p1 = torch.zeros((64, 64), dtype=torch.float16, device=DEV)
        torch.cuda.synchronize()
        fq.fq_w4a4_linear(qa64, sa64, qwp, swp, p1)
        if sync:
            torch.cuda.synchronize()
        q, s = fq.transform_quant(x, n1, n2, p1, e2, 0.9)
        torch.cuda.synchronize()
        res.append((q, s))
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])


# ------------------------------------------------------------------ binding shape checks
def test_binding_rejects_layouts_the_abi_cannot_express():
    n1 = n2 = 64
    K, T, N = n1 * n2, 8, 64
    big = torch.zeros((T, 2 * K), dtype=torch.float16, device=DEV)
    p = torch.eye(64, dtype=torch.float16, device=DEV)
    qw = torch.zeros((N, K // 2), dtype=torch.uint8, device=DEV)
    sw = torch.ones((N,), dtype=torch.float32, device=DEV)
    with pytest.raises(ValueError):                  # column slice of a fused projection: strided rows
        fq.flatquant_linear(big[:, :K], n1, n2, p, p, 0.9, qw, sw)
    qa = torch.zeros((T, K // 2), dtype=torch.uint8, device=DEV)
    sa = torch.ones((T,), dtype=torch.float32, device=DEV)
    with pytest.raises(ValueError):                  # output smaller than [T, N]
        fq.fq_w4a4_linear(qa, sa, qw, sw, torch.empty((T, N // 2), dtype=torch.float16, device=DEV))
    with pytest.raises(ValueError):                  # K mismatch between activations and weights
        fq.fq_w4a4_linear(qa, sa, qw[:, : K // 4], sw, torch.empty((T, N), dtype=torch.float16, device=DEV))
    with pytest.raises(ValueError):                  # non-contiguous weights
        fq.w4a4_gemm_i32(qa, torch.zeros((K // 2, N), dtype=torch.uint8, device=DEV).t())
    with pytest.raises(ValueError):                  # scale buffer of the wrong length
        fq.fq_transform_quant(big[:, :K], n1, n2, p, p, 0.9, qa, sa[:4])


def test_pdl_chains_and_shared_workspace_match_synchronised_runs():
    """The PDL protocol (a kernel lets dependents launch only after its own wait; inputs/outputs
    checked against the predecessor): (i) a chain GEMM -> independent transform -> transform
    whose P1 is the GEMM's output; (ii) one workspace reused by two linears (write-after-read:
    the second transform overwrites codes the first GEMM reads); (iii) independent linears
    back to back (transforms that start before the previous GEMM finishes).  Every result equals
    the same calls with a device synchronisation after each one."""
    n1 = n2 = 64
    K = n1 * n2
    e = torch.eye(64, dtype=torch.float16, device=DEV)
    qa0, sa0 = fq.transform_quant(torch.from_numpy(synth.activations(64, K, seed=20)).to(DEV), n1, n2, e, e, 0.9)
    qwp, swp = fq.transform_quant(torch.from_numpy(synth.weights(64, K, seed=21)).to(DEV), n1, n2, e, e, 1.0)
    xs = [torch.from_numpy(synth.activations(1500, K, seed=22 + i)).to(DEV) for i in range(3)]
    ws = [fq.transform_quant(torch.from_numpy(synth.weights(3072, K, seed=30 + i)).to(DEV), n1, n2, e, e, 1.0)
          for i in range(3)]
    torch.cuda.synchronize()

    def run(sync):
        def s():
            if sync:
                torch.cuda.synchronize()
        out = {}
        p1 = torch.zeros((64, 64), dtype=torch.float16, device=DEV)
        fq.fq_w4a4_linear(qa0, sa0, qwp, swp, p1); s()                        # (i) GEMM writes P1
        out["b"] = fq.transform_quant(xs[0], n1, n2, e, e, 0.9); s()          # independent transform
        out["c"] = fq.transform_quant(xs[1], n1, n2, p1, e, 0.9); s()         # reads the GEMM's output
        q_ws = torch.empty((1500, K // 2), dtype=torch.uint8, device=DEV)     # (ii) shared workspace
        s_ws = torch.empty((1500,), dtype=torch.float32, device=DEV)
        ys = []
        for i in range(2):
            fq.fq_transform_quant(xs[i], n1, n2, e, e, 0.9, q_ws, s_ws); s()
            ys.append(fq.w4a4_linear(q_ws, s_ws, *ws[i])); s()
        out["ws"] = ys
        outs = []                                                              # (iii) independent linears
        for i in range(3):
            q, sc = fq.transform_quant(xs[i], n1, n2, e, e, 0.9); s()
            outs.append(fq.w4a4_linear(q, sc, *ws[i])); s()
        out["ind"] = outs
        torch.cuda.synchronize()
        return out

    ref, got = run(True), run(False)
    for k in ("b", "c"):
        assert all(torch.equal(a, b) for a, b in zip(ref[k], got[k])), k
    for a, b in zip(ref["ws"] + ref["ind"], got["ws"] + got["ind"]):
        assert torch.equal(a, b)
