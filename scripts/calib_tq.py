"""Calibration of the transform kernel's timing at C3 size (T = 2048, 64 x 64):
event overhead of an empty launch, event-timed copies of the same byte count, the transform
alone / back to back / in-step marginal (step minus a GEMM-only step).  Prints JSON lines."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09426_b200 as fq  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
fq.load()
st = torch.cuda.current_stream()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)


def timed(fn, reps=30, do_flush=True):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        if do_flush:
            flush.zero_()
            flush.sum()
        torch.cuda._sleep(300_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return {"mean_us": round(sum(ts) / len(ts), 2), "median_us": round(ts[len(ts) // 2], 2), "min_us": round(ts[0], 2)}


def out(**kw):
    print(json.dumps(kw), flush=True)


one = torch.zeros(1, device=dev)
out(what="empty (1-element add)", **timed(lambda: one.add_(1), do_flush=False))
for mb in (8.4, 16.8, 64.0):
    n = int(mb * 1e6 / 2)
    a = torch.randn(n, device=dev).half()
    b = torch.empty_like(a)
    r = timed(lambda: b.copy_(a))
    out(what=f"copy {mb} MB -> {mb} MB", gbs=round(2 * n * 2 / (r["mean_us"] * 1e-6) / 1e9, 1), **r)

cfg = synth.config(os.environ.get("CFG", "C3"))
T = int(os.environ.get("T", cfg["T"]))
for lin in cfg["linears"]:
    x = torch.from_numpy(synth.activations(T, lin.K, seed=1, tag=lin.name)).to(dev)
    p1 = torch.from_numpy(synth.well_conditioned(lin.n1, seed=0, tag="p1")).to(dev)
    p2 = torch.from_numpy(synth.well_conditioned(lin.n2, seed=0, tag="p2")).to(dev)
    q = torch.empty((T, lin.K // 2), dtype=torch.uint8, device=dev)
    s = torch.empty((T,), device=dev)
    nbytes = T * (2 * lin.K + lin.K // 2 + 4)
    r = timed(lambda: fq.fq_transform_quant(x, lin.n1, lin.n2, p1, p2, 0.9, q, s))
    out(what=f"tq {lin.name} {lin.n1}x{lin.n2} T={T}", gbs=round(nbytes / (r["mean_us"] * 1e-6) / 1e9, 1), **r)
    # R back-to-back launches over distinct inputs (> L2 in total), PDL between them
    R = 8
    xs = [torch.from_numpy(synth.activations(T, lin.K, seed=10 + i, tag=lin.name)).to(dev) for i in range(R)]
    qs = [torch.empty_like(q) for _ in range(R)]
    ss = [torch.empty_like(s) for _ in range(R)]

    def chain():
        for i in range(R):
            fq.fq_transform_quant(xs[i], lin.n1, lin.n2, p1, p2, 0.9, qs[i], ss[i])
    r = timed(chain)
    out(what=f"tq x{R} back-to-back {lin.name}", per_launch_us=round(r["mean_us"] / R, 2),
        gbs=round(R * nbytes / (r["mean_us"] * 1e-6) / 1e9, 1), **r)
    del xs, qs, ss
