"""Launch gaps between back-to-back kernels (instrumented build): stamp->stamp, stamp->TQ->stamp."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FQ_TRACE_LIB"] = "1"
import paper_2410_09426_b200 as fq  # noqa: E402
import synth  # noqa: E402

lib = fq.load()
dev = torch.device("cuda:0")
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
st = (ctypes.c_ulonglong * 8)()
for _ in range(3):
    torch.cuda._sleep(100_000)
    lib.fq_debug_stamp(0, sp)
    lib.fq_debug_stamp(1, sp)
    lib.fq_debug_stamp(2, sp)
    torch.cuda.synchronize()
lib.fq_debug_stamps(st)
print(f"stamp->stamp gaps: {(st[1] - st[0]) / 1e3:.2f} us, {(st[2] - st[1]) / 1e3:.2f} us")
