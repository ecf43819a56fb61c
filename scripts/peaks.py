"""Reference tensor throughputs on this GPU: cuBLAS bf16 and int8 (torch._int_mm) GEMMs and our
W4A4 GEMM on the same square shape (burst: best of N after warm-up, CUDA events)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09426_b200 as fq  # noqa: E402

dev = torch.device("cuda:0")


def bench(fn, iters=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


for M, N, K in [(8192, 8192, 8192), (2048, 28672, 4096), (2048, 4096, 14336), (2048, 6144, 4096), (2048, 4096, 4096)]:
    ops = 2 * M * N * K
    xa = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
    wb = torch.randn(N, K, device=dev, dtype=torch.bfloat16)
    t_bf = bench(lambda: torch.matmul(xa, wb.t()))
    a8 = torch.randint(-8, 8, (M, K), device=dev, dtype=torch.int8)
    b8 = torch.randint(-8, 8, (K, N), device=dev, dtype=torch.int8).t().contiguous().t()
    try:
        t_i8 = bench(lambda: torch._int_mm(a8, b8))
    except Exception as e:  # noqa: BLE001
        t_i8 = float("nan")
        print("int_mm failed:", e)
    qa = torch.randint(0, 256, (M, K // 2), device=dev, dtype=torch.uint8)
    qw = torch.randint(0, 256, (N, K // 2), device=dev, dtype=torch.uint8)
    sa = torch.rand(M, device=dev) + 0.5
    sw = torch.rand(N, device=dev) + 0.5
    y = torch.empty(M, N, device=dev, dtype=torch.float16)
    t_w4 = bench(lambda: fq.fq_w4a4_linear(qa, sa, qw, sw, y))
    print(f"M={M} N={N} K={K}: cuBLAS bf16 {ops / t_bf / 1e9:7.1f} TFLOP/s | cuBLAS int8 (_int_mm) "
          f"{ops / t_i8 / 1e9:7.1f} TOPS | ours W4A4 {ops / t_w4 / 1e9:7.1f} TOPS")
