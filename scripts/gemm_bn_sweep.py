"""Pair-GEMM tile-width sweep: fq_w4a4_linear at T = 2048 on the C2/C3 shapes, L2 clean-flushed
before every timed launch (mean of event-timed launches).  FQ_PAIR_BN forces the width.
usage: FQ_PAIR_BN=96 python scripts/gemm_bn_sweep.py --tag bn96"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09426_b200 as fq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=2048)
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--tag", default="")
args = ap.parse_args()
dev = torch.device("cuda:0")
fq.load()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
g = torch.Generator(device=dev).manual_seed(0)
T = args.T
for name, N, K in (("qkv", 6144, 4096), ("o_proj", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)):
    qa = torch.randint(0, 256, (T, K // 2), generator=g, device=dev, dtype=torch.int32).to(torch.uint8)
    qw = torch.randint(0, 256, (N, K // 2), generator=g, device=dev, dtype=torch.int32).to(torch.uint8)
    sa = torch.rand(T, generator=g, device=dev) + 0.5
    sw = torch.rand(N, generator=g, device=dev) + 0.5
    y = torch.empty((T, N), dtype=torch.float16, device=dev)
    for _ in range(3):
        fq.fq_w4a4_linear(qa, sa, qw, sw, y)
    ts = []
    for _ in range(args.iters):
        flush.zero_()
        flush.sum()
        torch.cuda._sleep(200_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fq.fq_w4a4_linear(qa, sa, qw, sw, y)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    us = sum(ts) / len(ts)
    print(json.dumps({"tag": args.tag, "bn": os.environ.get("FQ_PAIR_BN", "auto"), "shape": name, "T": T, "N": N,
                      "K": K, "us_mean": round(us, 2), "tops": round(2 * T * N * K / us / 1e6, 1)}), flush=True)
