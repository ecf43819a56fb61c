"""Wide transform (C5 down_proj 128 x 224) launch time, L2 flushed: python scripts/wide_time.py [--T 32768]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09426_b200 as fq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=32768)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
dev = torch.device("cuda:0")
n1, n2 = 128, 224
x = torch.randn((a.T, n1 * n2), device=dev).half()
p1 = torch.linalg.qr(torch.randn(n1, n1, device=dev))[0].half().contiguous()
p2 = torch.linalg.qr(torch.randn(n2, n2, device=dev))[0].half().contiguous()
q = torch.empty((a.T, n1 * n2 // 2), dtype=torch.uint8, device=dev)
s = torch.empty(a.T, device=dev)
flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)
for _ in range(2):
    fq.fq_transform_quant(x, n1, n2, p1, p2, 0.9, q, s)
tot = 0.0
for _ in range(a.reps):
    flush.zero_()
    flush.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fq.fq_transform_quant(x, n1, n2, p1, p2, 0.9, q, s)
    e1.record()
    torch.cuda.synchronize()
    tot += e0.elapsed_time(e1)
us = tot / a.reps * 1e3
flops = 2 * a.T * n1 * n2 * (n1 + n2)
print(json.dumps({"T": a.T, "us": round(us, 1), "tflops": round(flops / (us * 1e-6) / 1e12, 1),
                  "gbs": round(a.T * (2 * n1 * n2 + n1 * n2 // 2 + 4) / (us * 1e-6) / 1e9, 1)}))
