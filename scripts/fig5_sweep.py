"""Decomposition sweep on the B200 (re-measures the kernel side of PAPER.md Fig. 5 / App. C.? at
PAPER.md:503, 525, 1270-1272): n = 4096 (LLaMA hidden size) and 14336 (LLaMA-3-8B intermediate)
split as n1 x n2, fused transform + quantize time per decomposition at prefill sizes, L2 flushed
(write + read) before every timed launch.  Shapes without a tensor-core kernel run the CUDA-core
fallback (reported as such); n1 x n2 with n2 > 256 is outside the ABI.
usage: python scripts/fig5_sweep.py [--T 2048 16384]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09426_b200 as fq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, nargs="+", default=[2048, 16384])
ap.add_argument("--iters", type=int, default=20)
args = ap.parse_args()
dev = torch.device("cuda:0")
fq.load()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
TC = {(64, 64), (64, 128), (80, 128), (96, 128), (112, 128), (128, 128), (128, 160), (128, 192), (128, 224),
      (128, 256)}
SPLITS = {4096: [(16, 256), (32, 128), (64, 64), (128, 32), (256, 16)],
          14336: [(56, 256), (64, 224), (112, 128), (128, 112), (224, 64)]}
for n, splits in SPLITS.items():
    for T in args.T:
        x = torch.randn((T, n), device=dev).half()
        q = torch.empty((T, n // 2), dtype=torch.uint8, device=dev)
        s = torch.empty(T, device=dev)
        for n1, n2 in splits:
            p1 = torch.linalg.qr(torch.randn(n1, n1, device=dev))[0].half()
            p2 = torch.linalg.qr(torch.randn(n2, n2, device=dev))[0].half()
            try:
                fq.fq_transform_quant(x, n1, n2, p1, p2, 0.9, q, s)
            except RuntimeError as e:
                print(json.dumps({"n": n, "n1": n1, "n2": n2, "T": T, "error": str(e)[:80]}), flush=True)
                continue
            ts = []
            for _ in range(args.iters):
                flush.zero_()
                flush.sum()
                torch.cuda._sleep(200_000)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fq.fq_transform_quant(x, n1, n2, p1, p2, 0.9, q, s)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            ts.sort()
            us = ts[len(ts) // 2]
            byts = T * (2 * n + n // 2 + 4) + 2 * (n1 * n1 + n2 * n2)
            print(json.dumps({"n": n, "n1": n1, "n2": n2, "T": T, "kernel": "tcgen05" if (n1, n2) in TC else "cuda-core/mma.sync",
                              "us": round(us, 2), "gbs": round(byts / us / 1e3, 1),
                              "tflops": round(2 * T * n * (n1 + n2) / us / 1e6, 1)}), flush=True)
