"""Device timeline of the tcgen05 transform kernel (instrumented build, -DFQ_TRACE).
usage: FQ_TRACE_LIB=1 python scripts/trace_tq.py --linear P_ug [--config C3]"""
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
ap.add_argument("--T", type=int, default=0, help="override the token count")
a = ap.parse_args()
cfg = synth.config(a.config)
lin = [l for l in cfg["linears"] if l.name == a.linear][0]
dev = torch.device("cuda:0")
T = a.T or cfg["T"]
x = torch.from_numpy(synth.activations(T, lin.K, seed=1, tag=lin.name)).to(dev)
p1 = torch.from_numpy(synth.well_conditioned(lin.n1, seed=0, tag="p1")).to(dev)
p2 = torch.from_numpy(synth.well_conditioned(lin.n2, seed=0, tag="p2")).to(dev)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for _ in range(3):
    flush.zero_()
    flush.sum()
    q, s = fq.transform_quant(x, lin.n1, lin.n2, p1, p2, 0.9)
torch.cuda.synchronize()
lib = fq.load()
buf = (ctypes.c_ulonglong * (4 * 256))()
lib.fq_debug_trace_tq(buf, 4 * 256)
tr = np.array(buf, dtype=np.int64).reshape(4, 256)
names = {0: "start", 1: "setup", 2: "pfull", 3: "pre_wait", 4: "post_wait", 120: "end(t0)", 121: "end(w4)", 122: "mma_loop_done", 123: "dealloc"}
for k in range(16):
    names[8 + k] = f"tma_issue[{k}]"
    names[24 + k] = f"mma1_xfull[{k}]"
    names[40 + k] = f"mma2_a2full[{k}]"
    names[56 + k] = f"epi_d1full[{k}]"
    names[72 + k] = f"epi1_done[{k}]"
    names[88 + k] = f"epi_d2full[{k}]"
    names[104 + k] = f"epi2_done[{k}]"
for k in range(8):
    for sub, nm in {1: "e1_ld", 2: "e1_xchg", 3: "e1_sts", 4: "e1_fence", 8: "e2_d2full", 9: "e2_ld", 10: "e2_xchg"}.items():
        names[128 + k * 16 + sub] = f"{nm}[{k}]"
t0 = tr[:, 0].min()
for cta in range(4):
    row = tr[cta]
    ev = sorted((int(row[i] - t0), names.get(i, str(i))) for i in range(256) if row[i] >= t0 and row[i] > 0)
    print(f"CTA {cta}: " + "  ".join(f"{n}@{t / 1000:.2f}us" for t, n in ev))

# ---- launch gaps: stamp kernel -> TQ kernel (all CTAs' start/end) -> stamp kernel ----
st = torch.cuda.current_stream()
sp = ctypes.c_void_p(st.cuda_stream)
for rep in range(3):
    flush.zero_()
    flush.sum()
    torch.cuda._sleep(200_000)
    lib.fq_debug_stamp(0, sp)
    fq.fq_transform_quant(x, lin.n1, lin.n2, p1, p2, 0.9, q, s)
    lib.fq_debug_stamp(1, sp)
    torch.cuda.synchronize()
stamps = (ctypes.c_ulonglong * 8)()
lib.fq_debug_stamps(stamps)
cta = (ctypes.c_ulonglong * 2048)()
lib.fq_debug_cta_tq(cta)
c = np.array(cta, dtype=np.int64).reshape(1024, 2)
ntiles = (T + (2 if lin.n1 == 64 else 1) - 1) // (2 if lin.n1 == 64 else 1)
c = c[: min(ntiles, 148)]
s0, s1 = stamps[0], stamps[1]
print(f"stamp0 -> first CTA start {(c[:, 0].min() - s0) / 1e3:.2f} us; last CTA start {(c[:, 0].max() - s0) / 1e3:.2f} us; "
      f"first CTA end {(c[:, 1].min() - s0) / 1e3:.2f} us; last CTA end {(c[:, 1].max() - s0) / 1e3:.2f} us; "
      f"stamp1 {(s1 - s0) / 1e3:.2f} us")
