"""Host-side cost of the Python binding + C-ABI enqueue for one linear at a decode size small
(T = 1, N = 512), enqueued behind a device sleep so the host time is the enqueue alone: is an
eager decode call host-bound, and what does the binding add to the raw ctypes call?"""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09426_b200 as fq  # noqa: E402
from paper_2410_09426_b200 import api  # noqa: E402

dev = torch.device("cuda:0")
T, n1, n2, N = 1, 64, 64, 512
K = n1 * n2
x_d = torch.randn(T, K, device=dev).half()
p1 = torch.eye(n1, dtype=torch.float16, device=dev)
p2 = torch.eye(n2, dtype=torch.float16, device=dev)
qw = torch.randint(0, 255, (N, K // 2), dtype=torch.uint8, device=dev)
sw = torch.rand(N, device=dev)
y_d = torch.empty(T, N, dtype=torch.float16, device=dev)
q = torch.empty(T, K // 2, dtype=torch.uint8, device=dev)
s = torch.empty(T, device=dev)
n = 300


def timed(label, fn):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)      # ~0.1 s: the device holds the queue, so host time is enqueue only
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{label:58s} host (enqueue only) {(t1 - t0) / n * 1e6:6.1f} us/call")


timed("fq_flatquant_linear (binding, current stream)",
      lambda: fq.fq_flatquant_linear(x_d, n1, n2, p1, p2, 0.9, qw, sw, y_d, q, s))
st = torch.cuda.current_stream()
timed("fq_flatquant_linear (binding, explicit stream)",
      lambda: fq.fq_flatquant_linear(x_d, n1, n2, p1, p2, 0.9, qw, sw, y_d, q, s, stream=st))
lib = api.load()
args = (x_d.data_ptr(), api._fq_dtype(x_d.dtype), T, n1, n2, p1.data_ptr(), p2.data_ptr(), 0.9, qw.data_ptr(),
        sw.data_ptr(), N, y_d.data_ptr(), api._fq_dtype(y_d.dtype), q.data_ptr(), s.data_ptr(), st.cuda_stream)
timed("raw ctypes fq_flatquant_linear", lambda: lib.fq_flatquant_linear(*args))
# the round-2 binding's pointer / stream marshalling, for comparison
old_ptr, old_stream = api._ptr, api._stream
api._ptr = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())
api._stream = lambda stream: ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
timed("fq_flatquant_linear (c_void_p marshalling, current stream)",
      lambda: fq.fq_flatquant_linear(x_d, n1, n2, p1, p2, 0.9, qw, sw, y_d, q, s))
api._ptr, api._stream = old_ptr, old_stream
