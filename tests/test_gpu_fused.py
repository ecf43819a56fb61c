"""GPU: the fused decode linear: at T <= 64 with n1 = n2 = 64,
fq_flatquant_linear runs the transform + quantize (Eq.3, 258-259, 367) inside the
decode GEMM launch, one kernel per linear, the codes meeting the GEMM in L2.

The fused kernel repeats the transform kernel's arithmetic operation for operation (same tcgen05
MMAs, same fp16 intermediate, same quantizer), so its codes, scales and outputs must be
BIT-IDENTICAL to fq_transform_quant followed by fq_w4a4_linear -- whose parity with the oracle is
established in test_gpu_parity.py -- and one end-to-end case is checked against the oracle too.
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

N1 = N2 = 64
K = N1 * N2


def _inputs(T, N, seed, out_dtype=torch.float16):
    x = torch.from_numpy(synth.activations(T, K, seed=seed, dtype=np.float32)).to(torch.float16).to(DEV)
    p1 = torch.from_numpy(synth.well_conditioned(N1, seed=seed, tag="p1", dtype=np.float32)).half().to(DEV)
    p2 = torch.from_numpy(synth.well_conditioned(N2, seed=seed, tag="p2", dtype=np.float32)).half().to(DEV)
    qw = torch.from_numpy(O.pack_int4(synth.random_codes(N, K, seed=seed, tag="qw"))).to(DEV)
    sw = torch.from_numpy(synth.random_scales(N, seed=seed, tag="sw")).to(DEV)
    return x, p1, p2, qw, sw


def _bufs(T, N, out_dtype=torch.float16):
    return (torch.empty((T, N), dtype=out_dtype, device=DEV),
            torch.full((T, K // 2), 0xAB, dtype=torch.uint8, device=DEV),
            torch.full((T,), -1.0, dtype=torch.float32, device=DEV))


def _two_kernels(x, p1, p2, alpha, qw, sw, out_dtype=torch.float16):
    """the unfused reference path: fq_transform_quant, then fq_w4a4_linear"""
    qa, sa = fq.transform_quant(x, N1, N2, p1, p2, alpha)
    y = fq.w4a4_linear(qa, sa, qw, sw, out_dtype=out_dtype)
    return y, qa, sa


def _fused(x, p1, p2, alpha, qw, sw, out_dtype=torch.float16, stream=None, bufs=None):
    T, N = x.shape[0], qw.shape[0]
    y, q, s = bufs if bufs is not None else _bufs(T, N, out_dtype)
    fq.fq_flatquant_linear(x, N1, N2, p1, p2, alpha, qw, sw, y, q, s, stream=stream)
    return y, q, s


@pytest.mark.parametrize("T", [1, 2, 3, 7, 16, 31, 32, 33, 47, 63, 64])
@pytest.mark.parametrize("N", [512, 4096, 6144, 28672])
def test_fused_decode_bit_identical_to_two_kernels(T, N):
    x, p1, p2, qw, sw = _inputs(T, N, seed=100 + T)
    n0 = fq.fq_launch_count()
    y, q, s = _fused(x, p1, p2, 0.9, qw, sw)
    assert fq.fq_launch_count() - n0 == 1                # one launch for the whole linear
    y2, q2, s2 = _two_kernels(x, p1, p2, 0.9, qw, sw)
    torch.cuda.synchronize()
    assert torch.equal(q, q2)
    assert torch.equal(s, s2)
    assert torch.equal(y, y2)


@pytest.mark.parametrize("out_dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("alpha", [1.0, 0.75])
def test_fused_decode_dtypes_and_clipping(out_dtype, alpha):
    T, N = 64, 4096
    x, p1, p2, qw, sw = _inputs(T, N, seed=7)
    y, q, s = _fused(x, p1, p2, alpha, qw, sw, out_dtype=out_dtype)
    y2, q2, s2 = _two_kernels(x, p1, p2, alpha, qw, sw, out_dtype=out_dtype)
    torch.cuda.synchronize()
    assert torch.equal(q, q2) and torch.equal(s, s2) and torch.equal(y, y2)


def test_fused_decode_vs_oracle():
    """end to end against the float64 oracle (same bars as the unfused chain tests)"""
    T, N = 64, 6144
    x = synth.activations(T, K, seed=3, tag="fused")
    p1 = synth.well_conditioned(N1, seed=3, tag="fused/p1")
    p2 = synth.well_conditioned(N2, seed=3, tag="fused/p2")
    w = synth.weights(N, K, seed=3, tag="fused")
    qw, sw, _ = O.prepare_weight(w, p1, p2, 1.0)
    sw32 = np.asarray(sw, np.float32)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
    y, q, s = _fused(dev(x), dev(p1), dev(p2), 0.9, dev(O.pack_int4(qw)), dev(sw32))
    torch.cuda.synchronize()
    qo, so, yo = O.transform_quant(x, p1, p2, 0.9)
    parity.check_transform(q.cpu().numpy(), s.cpu().numpy(), None, yo, qo, so, label="fused transform")
    out_o = O.w4a4_linear(qo, so, qw, sw32.astype(np.float64))
    out_same = O.w4a4_linear(O.unpack_int4(q.cpu().numpy()), s.cpu().numpy().astype(np.float64), qw,
                             sw32.astype(np.float64))
    parity.check_output(y.float().cpu().numpy(), out_o, out_same, label="fused output")


def test_fused_decode_back_to_back_shared_workspace_and_chain():
    """consecutive fused launches on one stream (PDL overlap): a shared q/s workspace (WAR/WAW
    on the codes) and a chain in which each linear reads the previous one's output (RAW)"""
    T, N = 48, 4096
    x, p1, p2, qw, sw = _inputs(T, N, seed=11)
    ws = _bufs(T, N)
    ys, refs = [], []
    xi = x
    for i in range(6):
        y = torch.empty((T, N), dtype=torch.float16, device=DEV)
        fq.fq_flatquant_linear(xi, N1, N2, p1, p2, 0.9, qw, sw, y, ws[1], ws[2])
        ys.append(y)
        xi = y if i % 2 == 0 else x                      # alternate: chained input / independent input
    xr = x
    for i in range(6):
        yr, _, _ = _two_kernels(xr, p1, p2, 0.9, qw, sw)
        refs.append(yr)
        xr = yr if i % 2 == 0 else x
    torch.cuda.synchronize()
    for a, b in zip(ys, refs):
        assert torch.equal(a, b)


def test_fused_decode_slot_reuse_and_graph_replay():
    """more fused launches than synchronisation slots (1024), and CUDA-graph replays that reuse
    the captured slots: every result stays bit-identical to the unfused path"""
    T, N = 64, 512
    x, p1, p2, qw, sw = _inputs(T, N, seed=5)
    ref, _, _ = _two_kernels(x, p1, p2, 0.9, qw, sw)
    bufs = _bufs(T, N)
    for _ in range(1100):
        _fused(x, p1, p2, 0.9, qw, sw, bufs=bufs)
    torch.cuda.synchronize()
    assert torch.equal(bufs[0], ref)
    s = torch.cuda.Stream()
    xs = x.clone()
    outs = [_bufs(T, N) for _ in range(3)]
    with torch.cuda.stream(s):
        _fused(xs, p1, p2, 0.9, qw, sw, stream=s, bufs=outs[0])      # warm-up outside capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for o in outs:
            _fused(xs, p1, p2, 0.9, qw, sw, stream=s, bufs=o)
    for seed in (21, 22, 23):
        xn, _, _, _, _ = _inputs(T, N, seed=seed)
        xs.copy_(xn)
        g.replay()
        torch.cuda.synchronize()
        r, _, _ = _two_kernels(xn, p1, p2, 0.9, qw, sw)
        torch.cuda.synchronize()
        for o in outs:
            assert torch.equal(o[0], r)


def test_fused_decode_not_taken_outside_its_shapes():
    """T > 64 keeps the two-kernel path (2 launches)"""
    T, N = 64, 512
    x, p1, p2, qw, sw = _inputs(T, N, seed=2)
    T2 = 65
    x2, _, _, _, _ = _inputs(T2, N, seed=2)
    y2, q2, s2 = _bufs(T2, N)
    n0 = fq.fq_launch_count()
    fq.fq_flatquant_linear(x2, N1, N2, p1, p2, 0.9, qw, sw, y2, q2, s2)
    assert fq.fq_launch_count() - n0 == 2
    torch.cuda.synchronize()


def test_fused_decode_concurrent_streams():
    """fused launches on three streams at once (each takes its own counter slot; the ticket CTAs
    are the lowest block indices of their grid, so they are resident whenever a spinning CTA is)"""
    T, N = 64, 6144
    x, p1, p2, qw, sw = _inputs(T, N, seed=31)
    ref, _, _ = _two_kernels(x, p1, p2, 0.9, qw, sw)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(3)]
    outs = [_bufs(T, N) for _ in range(9)]
    for i, o in enumerate(outs):
        _fused(x, p1, p2, 0.9, qw, sw, stream=streams[i % 3], bufs=o)
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o[0], ref)


def _inputs_g(T, N, n1, n2, seed):
    x = torch.from_numpy(synth.activations(T, n1 * n2, seed=seed, dtype=np.float32)).half().to(DEV)
    p1 = torch.from_numpy(synth.well_conditioned(n1, seed=seed, tag="p1", dtype=np.float32)).half().to(DEV)
    p2 = torch.from_numpy(synth.well_conditioned(n2, seed=seed, tag="p2", dtype=np.float32)).half().to(DEV)
    qw = torch.from_numpy(O.pack_int4(synth.random_codes(N, n1 * n2, seed=seed, tag="qw"))).to(DEV)
    sw = torch.from_numpy(synth.random_scales(N, seed=seed, tag="sw")).to(DEV)
    return x, p1, p2, qw, sw


@pytest.mark.parametrize("T", [1, 2, 5, 17, 32, 63, 64])
@pytest.mark.parametrize("N", [8192, 10240])
def test_fused_decode_64x128_bit_identical(T, N):
    """n = 8192 = 64 x 128 (the 70B models' hidden size): two tokens per ticket tile as two M = 128
    stage-1 groups, the phase-A tile over the first packed ring stages"""
    n1, n2 = 64, 128
    x, p1, p2, qw, sw = _inputs_g(T, N, n1, n2, seed=500 + T)
    y = torch.empty((T, N), dtype=torch.float16, device=DEV)
    q = torch.full((T, n1 * n2 // 2), 0xAB, dtype=torch.uint8, device=DEV)
    s = torch.full((T,), -1.0, dtype=torch.float32, device=DEV)
    n0 = fq.fq_launch_count()
    fq.fq_flatquant_linear(x, n1, n2, p1, p2, 0.9, qw, sw, y, q, s)
    assert fq.fq_launch_count() - n0 == 1
    q2, s2 = fq.transform_quant(x, n1, n2, p1, p2, 0.9)
    y2 = fq.w4a4_linear(q2, s2, qw, sw)
    torch.cuda.synchronize()
    assert torch.equal(q, q2) and torch.equal(s, s2) and torch.equal(y, y2)


@pytest.mark.parametrize("T", [1, 2, 5, 17, 32, 63, 64])
@pytest.mark.parametrize("N", [4096, 5120])
def test_fused_decode_112x128_bit_identical(T, N):
    """LLaMA-3-8B down_proj (14336 = 112 x 128): one token per ticket tile, the phase-A tile over
    the first packed ring stages (the ticket CTAs load their weights after it)"""
    n1, n2 = 112, 128
    x, p1, p2, qw, sw = _inputs_g(T, N, n1, n2, seed=200 + T)
    y = torch.empty((T, N), dtype=torch.float16, device=DEV)
    q = torch.full((T, n1 * n2 // 2), 0xAB, dtype=torch.uint8, device=DEV)
    s = torch.full((T,), -1.0, dtype=torch.float32, device=DEV)
    n0 = fq.fq_launch_count()
    fq.fq_flatquant_linear(x, n1, n2, p1, p2, 0.9, qw, sw, y, q, s)
    assert fq.fq_launch_count() - n0 == 1
    q2, s2 = fq.transform_quant(x, n1, n2, p1, p2, 0.9)
    y2 = fq.w4a4_linear(q2, s2, qw, sw)
    torch.cuda.synchronize()
    assert torch.equal(q, q2) and torch.equal(s, s2) and torch.equal(y, y2)


def test_fused_decode_112x128_chain_with_64x64():
    """a decode layer's linears back to back (64 x 64 and 112 x 128 fused launches, PDL overlap,
    shared workspace) equal the synchronised two-kernel results"""
    T = 64
    shapes = [(64, 64, 6144), (64, 64, 4096), (64, 64, 28672), (112, 128, 4096)]
    ins = [_inputs_g(T, N, n1, n2, seed=300 + i) for i, (n1, n2, N) in enumerate(shapes)]
    kmax = max(n1 * n2 for n1, n2, _ in shapes)
    qws = torch.empty((T, kmax // 2), dtype=torch.uint8, device=DEV)
    sws = torch.empty((T,), dtype=torch.float32, device=DEV)
    ys = []
    for (n1, n2, N), (x, p1, p2, qw, sw) in zip(shapes, ins):
        y = torch.empty((T, N), dtype=torch.float16, device=DEV)
        qv = qws.view(-1)[: T * n1 * n2 // 2].view(T, n1 * n2 // 2)     # one workspace for all linears
        fq.fq_flatquant_linear(x, n1, n2, p1, p2, 0.9, qw, sw, y, qv, sws)
        ys.append(y)
    torch.cuda.synchronize()
    for (n1, n2, N), (x, p1, p2, qw, sw), y in zip(shapes, ins, ys):
        q2, s2 = fq.transform_quant(x, n1, n2, p1, p2, 0.9)
        torch.cuda.synchronize()
        y2 = fq.w4a4_linear(q2, s2, qw, sw)
        torch.cuda.synchronize()
        assert torch.equal(y, y2)


@pytest.mark.parametrize("n1,n2,N", [(64, 64, 4096), (112, 128, 4096), (64, 128, 8192)])
@pytest.mark.parametrize("T", [1, 9, 64])
@pytest.mark.parametrize("p2_scale", [1.0, 1e5])
def test_fused_decode_bf16_bit_identical(n1, n2, N, T, p2_scale):
    """bf16 activations and transforms: P2 is scaled by a power of two into fp16 range inside the
    fused kernel as in the transform kernel (also for a P2 beyond fp16 range)"""
    x, p1, p2, qw, sw = _inputs_g(T, N, n1, n2, seed=400 + T)
    x, p1 = x.bfloat16(), p1.bfloat16()
    p2 = (p2.float() * p2_scale).bfloat16()
    y = torch.empty((T, N), dtype=torch.bfloat16, device=DEV)
    q = torch.full((T, n1 * n2 // 2), 0xAB, dtype=torch.uint8, device=DEV)
    s = torch.full((T,), -1.0, dtype=torch.float32, device=DEV)
    n0 = fq.fq_launch_count()
    fq.fq_flatquant_linear(x, n1, n2, p1, p2, 0.9, qw, sw, y, q, s)
    assert fq.fq_launch_count() - n0 == 1
    q2, s2 = fq.transform_quant(x, n1, n2, p1, p2, 0.9)
    y2 = fq.w4a4_linear(q2, s2, qw, sw, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    assert torch.equal(q, q2) and torch.equal(s, s2) and torch.equal(y, y2)


@pytest.mark.parametrize("T,N,fused", [(64, 128, False), (64, 256, False), (16, 128, True),
                                       (1, 65536, False), (64, 65536, False), (64, 37888, True)])
def test_fused_decode_falls_back_outside_its_limits(T, N, fused):
    """one CTA per tile and the whole grid resident at once (the GEMM CTAs wait for the ticket
    CTAs): outside that the linear runs the two kernels, with the same bits"""
    x, p1, p2, qw, sw = _inputs(T, N, seed=900 + T)
    n0 = fq.fq_launch_count()
    y, q, s = _fused(x, p1, p2, 0.9, qw, sw)
    assert fq.fq_launch_count() - n0 == (1 if fused else 2)
    y2, q2, s2 = _two_kernels(x, p1, p2, 0.9, qw, sw)
    torch.cuda.synchronize()
    assert torch.equal(q, q2)
    assert torch.equal(s, s2)
    assert torch.equal(y, y2)
