"""Decode (C4) step variants, L2 flushed before each: GEMM-only chain, two-kernel step, fused step,
and every linear alone fused vs two kernels; the GEMM-only chain is timed again after the fused
launches.  usage: python scripts/fused_probe.py [--reps 30]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09426_b200 as fq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--reps", type=int, default=30)
a = ap.parse_args()
dev = torch.device("cuda:0")
cfg = synth.config(a.config)
T = cfg["T"]
L = []
for lin in cfg["linears"]:
    x = torch.from_numpy(synth.activations(T, lin.K, seed=1000, tag=lin.name)).to(dev)
    p1 = torch.from_numpy(synth.well_conditioned(lin.n1, seed=0, tag=lin.name + "/p1")).to(dev)
    p2 = torch.from_numpy(synth.well_conditioned(lin.n2, seed=0, tag=lin.name + "/p2")).to(dev)
    w = torch.from_numpy(synth.weights(lin.N, lin.K, seed=0, tag=lin.name)).to(dev)
    qw, sw = fq.prepare_weight(w, lin.n1, lin.n2, p1, p2, 1.0)
    L.append(dict(lin=lin, x=x, p1=p1, p2=p2, qw=qw, sw=sw, q=torch.empty((T, lin.K // 2), dtype=torch.uint8, device=dev),
                  s=torch.empty((T,), device=dev), y=torch.empty((T, lin.N), dtype=torch.float16, device=dev)))
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
fs = torch.empty((), device=dev)
st = torch.cuda.current_stream()


def tq(d):
    fq.fq_transform_quant(d["x"], d["lin"].n1, d["lin"].n2, d["p1"], d["p2"], 0.9, d["q"], d["s"])


def gemm(d):
    fq.fq_w4a4_linear(d["q"], d["s"], d["qw"], d["sw"], d["y"])


def fused(d):
    fq.fq_flatquant_linear(d["x"], d["lin"].n1, d["lin"].n2, d["p1"], d["p2"], 0.9, d["qw"], d["sw"], d["y"], d["q"], d["s"])


def timed(fn):
    fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(a.reps):
        flush.zero_()
        torch.sum(flush, dim=0, out=fs)
        torch.cuda._sleep(300_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return round(tot / a.reps * 1e3, 2)


res = {}
res["gemm_only_before"] = timed(lambda: [gemm(d) for d in L])
res["two_kernel_step"] = timed(lambda: [(tq(d), gemm(d)) for d in L])
res["fused_step"] = timed(lambda: [fused(d) for d in L])
res["gemm_only_after"] = timed(lambda: [gemm(d) for d in L])
for d in L:
    n = d["lin"].name
    res[f"{n}_two_kernels"] = timed(lambda d=d: (tq(d), gemm(d)))
    res[f"{n}_fused"] = timed(lambda d=d: fused(d))
    res[f"{n}_gemm_only"] = timed(lambda d=d: gemm(d))
print(json.dumps(res))
