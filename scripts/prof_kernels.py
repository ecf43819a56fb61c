"""Run one linear of a config a few times (for ncu captures): transform_quant then w4a4_linear."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09426_b200 as fq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--linear", default="P_ug")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--gemm-impl", type=int, default=0)
ap.add_argument("--fused", action="store_true", help="fq_flatquant_linear (the fused decode linear at T <= 64)")
a = ap.parse_args()
cfg = synth.config(a.config)
lin = [l for l in cfg["linears"] if l.name == a.linear][0]
dev = torch.device("cuda:0")
T = cfg["T"]
x = torch.from_numpy(synth.activations(T, lin.K, seed=1, tag=lin.name)).to(dev)
p1 = torch.from_numpy(synth.well_conditioned(lin.n1, seed=0, tag="p1")).to(dev)
p2 = torch.from_numpy(synth.well_conditioned(lin.n2, seed=0, tag="p2")).to(dev)
qw = torch.from_numpy(synth.random_codes(lin.N, lin.K // 2, seed=0).view(np.uint8)).to(dev)
sw = torch.from_numpy(synth.random_scales(lin.N)).to(dev)
fq.fq_set_gemm_impl(a.gemm_impl)
for _ in range(a.iters):
    if a.fused:
        y = fq.flatquant_linear(x, lin.n1, lin.n2, p1, p2, 0.9, qw, sw)
        continue
    q, s = fq.transform_quant(x, lin.n1, lin.n2, p1, p2, 0.9)
    y = fq.w4a4_linear(q, s, qw, sw)
torch.cuda.synchronize()
print("done", a.config, lin)
