"""One small launch of every product kernel (transform: tcgen05 64x64, 112x128, wide 128x224, asym,
P2 = I, SMALL decode config; GEMM: pair kernel sym/asym, decode kernel; the fused decode linear;
KV quant) for compute-sanitizer runs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2410_09426_b200 as fq  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


for n1, n2, T in [(64, 64, 300), (112, 128, 150), (128, 224, 40), (32, 128, 64)]:
    x = t(synth.activations(T, n1 * n2, seed=1))
    p1 = t(synth.well_conditioned(n1, seed=1, tag="p1"))
    p2 = None if (n1, n2) == (32, 128) else t(synth.well_conditioned(n2, seed=1, tag="p2"))
    q, s = fq.transform_quant(x, n1, n2, p1, p2, 0.9)
    if p2 is not None and (n1, n2) != (128, 224):
        fq.transform_quant_asym(x, n1, n2, p1, p2, 0.9)
torch.cuda.synchronize()
for T, N, K in [(300, 520, 4096), (40, 776, 2048)]:
    qa = t(O.pack_int4(synth.random_codes(T, K, seed=2)))
    qw = t(O.pack_int4(synth.random_codes(N, K, seed=3)))
    sa = t(synth.random_scales(T, seed=2))
    sw = t(synth.random_scales(N, seed=3))
    fq.w4a4_linear(qa, sa, qw, sw)
    za = torch.zeros((T,), dtype=torch.int8, device=dev)
    fq.w4a4_linear(qa, sa, qw, sw, za=za, colsum_w=fq.weight_colsum(qw))
# fused decode linear (transform inside the decode GEMM launch) and the SMALL decode transform
for T, N in [(40, 1024), (7, 512)]:
    x = t(synth.activations(T, 4096, seed=5))
    p1 = t(synth.well_conditioned(64, seed=5, tag="p1"))
    p2 = t(synth.well_conditioned(64, seed=5, tag="p2"))
    qw = t(O.pack_int4(synth.random_codes(N, 4096, seed=6)))
    sw = t(synth.random_scales(N, seed=6))
    fq.flatquant_linear(x, 64, 64, p1, p2, 0.9, qw, sw)
x = t(synth.activations(20, 112 * 128, seed=7))
fq.transform_quant(x, 112, 128, t(synth.well_conditioned(112, seed=7, tag="p1")), t(synth.well_conditioned(128, seed=7, tag="p2")), 0.9)
torch.cuda.synchronize()
kv = t(synth.activations(256, 128, seed=4, pivot_channels=0))
fq.kv_quant(kv, t(synth.well_conditioned(128, seed=4, tag="ph")), 0.95)
torch.cuda.synchronize()
print("sanitize_small done")
