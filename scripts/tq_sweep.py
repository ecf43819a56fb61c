"""Transform+quant kernel duration vs token count (CUDA events, L2 flushed before each launch):
the slope is the per-tile cost, the intercept the fixed (launch + prologue + drain) cost.
usage: python scripts/tq_sweep.py [--impl 0|1] [--shapes 64x64,112x128]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09426_b200 as fq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--impl", type=int, default=0)
ap.add_argument("--shapes", default="64x64,64x128,112x128")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--T", default="148,296,592,1184,2048,2368,4736,9472,18944,32768")
ap.add_argument("--ncu", action="store_true", help="one launch per T (for ncu captures)")
a = ap.parse_args()
dev = torch.device("cuda:0")
fq.fq_set_tq_impl(a.impl)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for shp in a.shapes.split(","):
    n1, n2 = map(int, shp.split("x"))
    n = n1 * n2
    p1 = torch.from_numpy(synth.well_conditioned(n1, seed=0, tag="p1")).to(dev)
    p2 = torch.from_numpy(synth.well_conditioned(n2, seed=0, tag="p2")).to(dev)
    print(f"# {n1}x{n2} impl {a.impl}")
    for T in map(int, a.T.split(",")):
        x = torch.from_numpy(synth.activations(T, n, seed=1)).to(dev)
        q = torch.empty((T, n // 2), dtype=torch.uint8, device=dev)
        s = torch.empty((T,), dtype=torch.float32, device=dev)
        ts = []
        for it in range(1 if a.ncu else a.iters + 3):
            flush.zero_()
            torch.cuda._sleep(200_000)       # keep the GPU busy while the host enqueues the launch
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fq.fq_transform_quant(x, n1, n2, p1, p2, 0.9, q, s)
            e1.record()
            torch.cuda.synchronize()
            if it >= 3 or a.ncu:
                ts.append(e0.elapsed_time(e1) * 1e3)
        us = float(np.median(ts))
        byts = T * (2 * n + n // 2 + 4)
        print(f"T={T:6d}  {us:8.2f} us  {byts / us / 1e3:8.1f} GB/s  ({byts / 6539.2e3:7.2f} us at HBM peak)")
