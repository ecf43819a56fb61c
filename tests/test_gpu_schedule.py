"""GPU: the per-launch counter slots of the transform kernel's dynamic tile schedule (round 2c,
DESIGN.md K1) -- every tile is transformed exactly once whatever the CTA placement, slots are
reset by each launch's last CTA (more launches than slots, CUDA-graph replays), and launches on
concurrent streams use their own slots.  Results are compared with the synchronised single-launch
result of the same kernel and, for one case, with the float64 oracle."""
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


def _inputs(T, n1, n2, seed):
    x = torch.from_numpy(synth.activations(T, n1 * n2, seed=seed, dtype=np.float32)).half().to(DEV)
    p1 = torch.from_numpy(synth.well_conditioned(n1, seed=seed, tag="p1", dtype=np.float32)).half().to(DEV)
    p2 = torch.from_numpy(synth.well_conditioned(n2, seed=seed, tag="p2", dtype=np.float32)).half().to(DEV)
    return x, p1, p2


@pytest.mark.parametrize("n1,n2,T", [(64, 64, 2048), (64, 64, 301), (112, 128, 1000), (64, 128, 777)])
def test_dynamic_schedule_matches_oracle_and_is_deterministic(n1, n2, T):
    x, p1, p2 = _inputs(T, n1, n2, seed=T)
    q1, s1 = fq.transform_quant(x, n1, n2, p1, p2, 0.9)
    q2, s2 = fq.transform_quant(x, n1, n2, p1, p2, 0.9)
    torch.cuda.synchronize()
    assert torch.equal(q1, q2) and torch.equal(s1, s2)
    rows = np.arange(0, T, max(1, T // 64))
    xo = x.float().cpu().numpy().astype(np.float64)[rows]
    qo, so, yo = O.transform_quant(xo, p1.float().cpu().numpy().astype(np.float64),
                                   p2.float().cpu().numpy().astype(np.float64), 0.9)
    parity.check_transform(q1.cpu().numpy()[rows], s1.cpu().numpy()[rows], None, yo, qo, so, label="dynamic schedule")


def test_dynamic_schedule_slot_reuse_graph_and_streams():
    n1, n2, T = 64, 64, 600
    x, p1, p2 = _inputs(T, n1, n2, seed=3)
    ref_q, ref_s = fq.transform_quant(x, n1, n2, p1, p2, 1.0)
    torch.cuda.synchronize()
    q = torch.empty_like(ref_q)
    s = torch.empty_like(ref_s)
    for _ in range(1100):                                  # more launches than the 1024 slots
        fq.fq_transform_quant(x, n1, n2, p1, p2, 1.0, q, s)
    torch.cuda.synchronize()
    assert torch.equal(q, ref_q) and torch.equal(s, ref_s)
    # two streams, interleaved launches, each with its own outputs
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [(torch.empty_like(ref_q), torch.empty_like(ref_s)) for _ in range(8)]
    for i, (qq, ss) in enumerate(outs):
        fq.fq_transform_quant(x, n1, n2, p1, p2, 1.0, qq, ss, stream=streams[i % 2])
    torch.cuda.synchronize()
    for qq, ss in outs:
        assert torch.equal(qq, ref_q) and torch.equal(ss, ref_s)
    # CUDA graph: the captured launches keep their slots; replays must reset them
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    xs = x.clone()
    gq = [(torch.empty_like(ref_q), torch.empty_like(ref_s)) for _ in range(3)]
    with torch.cuda.stream(st):
        fq.fq_transform_quant(xs, n1, n2, p1, p2, 1.0, gq[0][0], gq[0][1], stream=st)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=st):
        for qq, ss in gq:
            fq.fq_transform_quant(xs, n1, n2, p1, p2, 1.0, qq, ss, stream=st)
    for seed in (11, 12, 13):
        xn, _, _ = _inputs(T, n1, n2, seed=seed)
        xs.copy_(xn)
        g.replay()
        torch.cuda.synchronize()
        rq, rs = fq.transform_quant(xn, n1, n2, p1, p2, 1.0)
        torch.cuda.synchronize()
        for qq, ss in gq:
            assert torch.equal(qq, rq) and torch.equal(ss, rs)


def test_dynamic_schedule_overlaps_a_preceding_gemm_correctly():
    """the transform of the next linear runs while the previous GEMM drains (PDL, disjoint
    buffers); chained and independent inputs give the synchronised results"""
    n1, n2, T, N = 64, 64, 2048, 4096
    x, p1, p2 = _inputs(T, n1, n2, seed=5)
    qw = torch.from_numpy(O.pack_int4(synth.random_codes(N, n1 * n2, seed=5))).to(DEV)
    sw = torch.from_numpy(synth.random_scales(N, seed=5)).to(DEV)
    ys = []
    xi = x
    for i in range(4):
        q, s = fq.transform_quant(xi, n1, n2, p1, p2, 0.9)
        y = fq.w4a4_linear(q, s, qw, sw)
        ys.append(y)
        xi = y if i % 2 == 0 else x
    torch.cuda.synchronize()
    xi = x
    for i in range(4):
        q, s = fq.transform_quant(xi, n1, n2, p1, p2, 0.9)
        torch.cuda.synchronize()
        y = fq.w4a4_linear(q, s, qw, sw)
        torch.cuda.synchronize()
        assert torch.equal(y, ys[i])
        xi = y if i % 2 == 0 else x
