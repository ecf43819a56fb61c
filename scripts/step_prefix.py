"""In-step cost of every kernel of a bench step: the step is timed with only its first k kernels
(k = 1 .. 2L, transform and GEMM of each linear in order; L2 flushed before each step), so the
increments are each kernel's marginal cost with PDL overlap included.  --config C3|C4."""
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
layers = []
for lin in cfg["linears"]:
    x = torch.from_numpy(synth.activations(T, lin.K, seed=1000, tag=lin.name)).to(dev)
    p1 = torch.from_numpy(synth.well_conditioned(lin.n1, seed=0, tag=lin.name + "/p1")).to(dev)
    p2 = torch.from_numpy(synth.well_conditioned(lin.n2, seed=0, tag=lin.name + "/p2")).to(dev)
    w = torch.from_numpy(synth.weights(lin.N, lin.K, seed=0, tag=lin.name)).to(dev)
    qw, sw = fq.prepare_weight(w, lin.n1, lin.n2, p1, p2, 1.0)
    layers.append((lin, x, p1, p2, qw, sw, torch.empty((T, lin.K // 2), dtype=torch.uint8, device=dev),
                   torch.empty((T,), device=dev), torch.empty((T, lin.N), dtype=torch.float16, device=dev)))
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
fs = torch.empty((), device=dev)
st = torch.cuda.current_stream()


def kernels():
    out = []
    for lin, x, p1, p2, qw, sw, q, s, y in layers:
        out.append((f"tq_{lin.name}", lambda lin=lin, x=x, p1=p1, p2=p2, q=q, s=s:
                    fq.fq_transform_quant(x, lin.n1, lin.n2, p1, p2, 0.9, q, s)))
        out.append((f"gemm_{lin.name}", lambda q=q, s=s, qw=qw, sw=sw, y=y: fq.fq_w4a4_linear(q, s, qw, sw, y)))
    return out


ks = kernels()
for _, f in ks:
    f()
torch.cuda.synchronize()
prev = 0.0
res = []
for k in range(0, len(ks) + 1):
    tot = 0.0
    for _ in range(a.reps):
        flush.zero_()
        torch.sum(flush, dim=0, out=fs)
        torch.cuda._sleep(300_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _, f in ks[:k]:
            f()
        e1.record(st)
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    t = tot / a.reps * 1e3
    res.append({"k": k, "last": ks[k - 1][0] if k else "(empty)", "prefix_us": round(t, 2), "delta_us": round(t - prev, 2)})
    prev = t
for r in res:
    print(json.dumps(r))
