"""W4A4 GEMM throughput on the config shapes (C3 linears, C2, 8192^3): R back-to-back launches
between two events (launch overhead amortised), best of several repetitions.  FQ_LIB selects an
experiment build.  Prints one JSON line per shape."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09426_b200 as fq  # noqa: E402

dev = torch.device("cuda:0")
fq.load()
R = 20
SHAPES = [("qkv", 2048, 6144, 4096), ("o_proj", 2048, 4096, 4096), ("gate_up", 2048, 28672, 4096),
          ("down", 2048, 4096, 14336), ("sq8192", 8192, 8192, 8192)]
tag = os.path.basename(os.environ.get("FQ_LIB", "default"))
IMPLS = [int(v) for v in os.environ.get("IMPLS", "0").split(",")]   # 3/4/5/7: tile width 192/160/128/256
for impl, (name, M, N, K) in [(i, sh) for sh in SHAPES for i in IMPLS]:
    fq.fq_set_gemm_impl(impl)
    qa = torch.randint(0, 256, (M, K // 2), device=dev, dtype=torch.uint8)
    qw = torch.randint(0, 256, (N, K // 2), device=dev, dtype=torch.uint8)
    sa = torch.rand(M, device=dev) + 0.5
    sw = torch.rand(N, device=dev) + 0.5
    y = torch.empty(M, N, device=dev, dtype=torch.float16)
    for _ in range(3):
        fq.fq_w4a4_linear(qa, sa, qw, sw, y)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(R):
            fq.fq_w4a4_linear(qa, sa, qw, sw, y)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / R)
    print(json.dumps({"lib": tag, "impl": impl, "shape": name, "M": M, "N": N, "K": K, "us": round(best * 1e3, 2),
                      "tops": round(2 * M * N * K / (best * 1e-3) / 1e12, 1)}), flush=True)
