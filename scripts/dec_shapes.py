"""Decode GEMM (T = 64) on the C4 shapes: R back-to-back launches between two events, L2 not
flushed (weights 12-59 MB partly L2-resident: a relative comparison of experiment builds)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09426_b200 as fq  # noqa: E402

dev = torch.device("cuda:0")
tag = os.path.basename(os.environ.get("FQ_LIB", "default"))
R = 20
for name, N, K in [("qkv", 6144, 4096), ("o_proj", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]:
    T = 64
    qa = torch.randint(0, 256, (T, K // 2), device=dev, dtype=torch.uint8)
    qws = [torch.randint(0, 256, (N, K // 2), device=dev, dtype=torch.uint8) for _ in range(4)]
    sa = torch.rand(T, device=dev) + 0.5
    sw = torch.rand(N, device=dev) + 0.5
    y = torch.empty(T, N, device=dev, dtype=torch.float16)
    for i in range(4):
        fq.fq_w4a4_linear(qa, sa, qws[i], sw, y)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)             # the host enqueues the launches ahead of the GPU
        a.record()
        for i in range(R):
            fq.fq_w4a4_linear(qa, sa, qws[i % 4], sw, y)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / R)
    print(json.dumps({"lib": tag, "shape": name, "us": round(best * 1e3, 2),
                      "gbs": round(N * K / 2 / (best * 1e-3) / 1e9, 1)}), flush=True)
