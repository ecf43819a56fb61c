"""Host-side cost of one fq_flatquant_linear_host_async call (Python binding + C ABI enqueue) and
of the device work it enqueues, at C4 (decode) shapes: is the e2e step host-bound?"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09426_b200 as fq  # noqa: E402
from paper_2410_09426_b200 import api  # noqa: E402

dev = torch.device("cuda:0")
T, n1, n2, N = 64, 64, 64, 28672
K = n1 * n2
x_h = torch.randn(T, K).half().pin_memory()
x_d = torch.empty(T, K, dtype=torch.float16, device=dev)
p1 = torch.eye(n1, dtype=torch.float16, device=dev)
p2 = torch.eye(n2, dtype=torch.float16, device=dev)
qw = torch.randint(0, 255, (N, K // 2), dtype=torch.uint8, device=dev)
sw = torch.rand(N, device=dev)
y_h = torch.empty(T, N, dtype=torch.float16).pin_memory()
y_d = torch.empty(T, N, dtype=torch.float16, device=dev)
q = torch.empty(T, K // 2, dtype=torch.uint8, device=dev)
s = torch.empty(T, device=dev)
st = torch.cuda.Stream()
for _ in range(10):
    fq.fq_flatquant_linear_host(x_h, x_d, n1, n2, p1, p2, 0.9, qw, sw, y_h, y_d, q, s, stream=st, sync=False)
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    fq.fq_flatquant_linear_host(x_h, x_d, n1, n2, p1, p2, 0.9, qw, sw, y_h, y_d, q, s, stream=st, sync=False)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"python call: {(t1 - t0) / n * 1e6:.1f} us host per call; device drained {(t2 - t0) / n * 1e6:.1f} us per call")
lib = api.load()
args = (api._ptr(x_h), api._ptr(x_d), api._fq_dtype(x_d.dtype), T, n1, n2, api._ptr(p1), api._ptr(p2), 0.9,
        api._ptr(qw), api._ptr(sw), N, api._ptr(y_h), api._ptr(y_d), api._fq_dtype(y_d.dtype), api._ptr(q),
        api._ptr(s), api._stream(st))
t0 = time.perf_counter()
for _ in range(n):
    lib.fq_flatquant_linear_host_async(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"raw ctypes call: {(t1 - t0) / n * 1e6:.1f} us host per call; device drained {(t2 - t0) / n * 1e6:.1f} us per call")
