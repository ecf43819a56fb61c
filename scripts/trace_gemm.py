"""Device timeline of the first CTA pair of the W4A4 GEMM (instrumented build, -DFQ_TRACE).
usage: python scripts/trace_gemm.py --linear P_ug"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FQ_TRACE_LIB"] = "1"
import paper_2410_09426_b200 as fq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--linear", default="P_ug")
a = ap.parse_args()
cfg = synth.config(a.config)
lin = [l for l in cfg["linears"] if l.name == a.linear][0]
dev = torch.device("cuda:0")
T, K, N = cfg["T"], lin.K, lin.N
qa = torch.randint(0, 256, (T, K // 2), device=dev, dtype=torch.uint8)
qw = torch.randint(0, 256, (N, K // 2), device=dev, dtype=torch.uint8)
sa = torch.rand(T, device=dev) + 0.5
sw = torch.rand(N, device=dev) + 0.5
y = torch.empty(T, N, device=dev, dtype=torch.float16)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for _ in range(3):
    flush.zero_()
    torch.cuda._sleep(100_000)
    fq.fq_w4a4_linear(qa, sa, qw, sw, y)
torch.cuda.synchronize()
lib = fq.load()
buf = (ctypes.c_ulonglong * 512)()
lib.fq_debug_trace_gemm(buf)
tr = np.array(buf, dtype=np.int64).reshape(2, 256)
t0 = tr[:, 250].min()
kb = (K + 127) // 128
print(f"{a.linear}: T={T} N={N} K={K}, {kb} k-blocks per tile")
for cta in range(2):
    r = tr[cta]
    rel = lambda i: (r[i] - t0) / 1e3  # noqa: E731
    conv = [rel(j) for j in range(64) if r[j] > 0]
    print(f"CTA {cta}: start {rel(250):.2f}  end {rel(251):.2f} us")
    print("  stage full signalled (conv): " + " ".join(f"{c:.2f}" for c in conv[:64]))
    if cta == 0:
        mma = [rel(64 + j) for j in range(64) if r[64 + j] > 0]
        print("  MMA full-wait done:          " + " ".join(f"{c:.2f}" for c in mma))
        print("  tile commit: " + " ".join(f"{rel(128 + i):.2f}" for i in range(8) if r[128 + i] > 0))
    print("  epi tfull:   " + " ".join(f"{rel(136 + i):.2f}" for i in range(8) if r[136 + i] > 0))
    print("  epi done:    " + " ".join(f"{rel(144 + i):.2f}" for i in range(8) if r[144 + i] > 0))
r = tr[0]
print("A thread (CTA0): job start -> [empty ok, packed-A ok, STTM+wait done, signalled] (us after start)")
for j in range(10):
    v = [r[160 + j * 5 + i] for i in range(5)]
    if v[0] > 0:
        print(f"  job {16 + j}: start {(v[0] - t0) / 1e3:.2f} us  +" + " +".join(f"{(x - v[0]) / 1e3:.3f}" for x in v[1:]))
print("B thread (CTA0): [waits done, STS done, fence done]")
for j in range(10):
    v = [r[210 + j * 3 + i] for i in range(3)]
    if v[0] > 0:
        print(f"  job {16 + j}: start {(v[0] - t0) / 1e3:.2f} us  +" + " +".join(f"{(x - v[0]) / 1e3:.3f}" for x in v[1:]))
