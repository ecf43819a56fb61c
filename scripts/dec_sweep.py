"""Decode GEMM sweep: fq_w4a4_linear at T tokens on the C4 (LLaMA-3-8B) shapes, L2 flushed
before every timed launch, CUDA events on the launching stream.  Prints one JSON line per shape.
usage: python scripts/dec_sweep.py [--T 64] [--iters 30]   (FQ_DEC_SPLIT / FQ_GEMM_IMPL env)"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09426_b200 as fq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=64)
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--tag", default="")
ap.add_argument("--only", default="", help="comma-separated shape names (qkv,o_proj,gate_up,down)")
ap.add_argument("--flush", default="clean", choices=["write", "clean", "rotate"],
                help="write: 256 MiB write before each launch (leaves dirty L2 lines); clean: write then "
                     "read 256 MiB (cold, clean L2); rotate: back-to-back launches over weight copies > 3x L2")
args = ap.parse_args()
dev = torch.device("cuda:0")
fq.load()
if os.environ.get("FQ_GEMM_IMPL"):
    fq.fq_set_gemm_impl(int(os.environ["FQ_GEMM_IMPL"]))
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
g = torch.Generator(device=dev).manual_seed(0)
T = args.T
for name, N, K in (("qkv", 6144, 4096), ("o_proj", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)):
    if args.only and name not in args.only.split(","):
        continue
    qa = torch.randint(0, 256, (T, K // 2), generator=g, device=dev, dtype=torch.int32).to(torch.uint8)
    qw = torch.randint(0, 256, (N, K // 2), generator=g, device=dev, dtype=torch.int32).to(torch.uint8)
    sa = torch.rand(T, generator=g, device=dev) + 0.5
    sw = torch.rand(N, generator=g, device=dev) + 0.5
    y = torch.empty((T, N), dtype=torch.float16, device=dev)
    for _ in range(3):
        fq.fq_w4a4_linear(qa, sa, qw, sw, y)
    ts = []
    if args.flush == "rotate":
        R = max(2, (3 * 126 * 2 ** 20) // qw.numel() + 1)
        qws = [qw.clone() for _ in range(R)]
        for _ in range(max(3, args.iters // 5)):
            torch.cuda._sleep(200_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for r in range(4 * R):
                fq.fq_w4a4_linear(qa, sa, qws[r % R], sw, y)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3 / (4 * R))
        del qws
    for _ in range(args.iters if args.flush != "rotate" else 0):
        flush.zero_()
        if args.flush == "clean":
            flush.sum()
        torch.cuda._sleep(200_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fq.fq_w4a4_linear(qa, sa, qw, sw, y)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    us = ts[len(ts) // 2]
    byts = T * K // 2 + N * K // 2 + 4 * (T + N) + 2 * T * N
    print(json.dumps({"tag": args.tag, "flush": args.flush, "shape": name, "T": T, "N": N, "K": K, "split": os.environ.get("FQ_DEC_SPLIT", "auto"),
                      "us_median": round(us, 2), "us_min": round(ts[0], 2), "gbs": round(byts / us / 1e3, 1)}), flush=True)
