"""Device timeline of the decode GEMM (instrumented build, -DFQ_TRACE): CTAs 0, 1 and the last
two of the last launch.  usage: python scripts/trace_dec.py [--N 4096 --K 4096 --T 64]"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FQ_TRACE_LIB"] = "1"
import paper_2410_09426_b200 as fq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=4096)
ap.add_argument("--K", type=int, default=4096)
ap.add_argument("--T", type=int, default=64)
ap.add_argument("--flush", action="store_true")
ap.add_argument("--fused", action="store_true", help="fq_flatquant_linear (fused decode linear, n1 = n2 = 64)")
a = ap.parse_args()
dev = torch.device("cuda:0")
T, K, N = a.T, a.K, a.N
qa = torch.randint(0, 256, (T, K // 2), device=dev, dtype=torch.uint8)
qws = [torch.randint(0, 256, (N, K // 2), device=dev, dtype=torch.uint8) for _ in range(4)]
sa = torch.rand(T, device=dev) + 0.5
sw = torch.rand(N, device=dev) + 0.5
y = torch.empty(T, N, device=dev, dtype=torch.float16)
xs = torch.randn(T, K, device=dev).half()
p1 = torch.linalg.qr(torch.randn(64, 64, device=dev))[0].half().contiguous()
p2 = torch.linalg.qr(torch.randn(64, 64, device=dev))[0].half().contiguous()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for i in range(8):
    if a.flush:
        flush.zero_()
        flush.sum()
        torch.cuda._sleep(100_000)
    if a.fused:
        fq.fq_flatquant_linear(xs, 64, 64, p1, p2, 0.9, qws[i % 4], sw, y, qa, sa)
    else:
        fq.fq_w4a4_linear(qa, sa, qws[i % 4], sw, y)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 512)()
fq.load().fq_debug_trace_dec(buf)
tr = np.array(buf, dtype=np.int64).reshape(4, 128)
t0 = tr[:, 0][tr[:, 0] > 0].min()
print(f"decode GEMM{' (fused)' if a.fused else ''} T={T} N={N} K={K} ({'flushed' if a.flush else 'back to back'}), "
      "us after the first CTA start")
for c in range(4):
    r = tr[c]
    if r[0] == 0:
        continue
    f = lambda i: f"{(r[i] - t0) / 1e3:.2f}" if r[i] > 0 else "-"  # noqa: E731
    print(f"CTA slot {c}: start {f(0)} setup {f(1)} tfull {f(112)} stored {f(113)} reduced {f(114)} end {f(115)}")
    if a.fused:
        print(f"  fused: X landed {f(116)} epi1 done {f(119)} MMA2 done {f(120)} stored {f(121)} fenced {f(122)} "
              f"tile counted {f(117)} all counted {f(118)}")
    print("  TMA issue  : " + " ".join(f(4 + j) for j in range(36) if r[4 + j] > 0))
    print("  conv done  : " + " ".join(f(40 + j) for j in range(36) if r[40 + j] > 0))
    print("  MMA issued : " + " ".join(f(76 + j) for j in range(36) if r[76 + j] > 0))
