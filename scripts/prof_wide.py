"""One wide-transform launch (C5 down_proj, 128 x 224) for ncu: python scripts/prof_wide.py [--T 32768]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09426_b200 as fq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=32768)
a = ap.parse_args()
dev = torch.device("cuda:0")
n1, n2 = 128, 224
x = torch.randn((a.T, n1 * n2), device=dev).half()
p1 = torch.linalg.qr(torch.randn(n1, n1, device=dev))[0].half()
p2 = torch.linalg.qr(torch.randn(n2, n2, device=dev))[0].half()
q = torch.empty((a.T, n1 * n2 // 2), dtype=torch.uint8, device=dev)
s = torch.empty(a.T, device=dev)
for _ in range(3):
    fq.fq_transform_quant(x, n1, n2, p1, p2, 0.9, q, s)
torch.cuda.synchronize()
