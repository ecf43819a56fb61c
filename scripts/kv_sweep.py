"""KV-cache quantization kernel sweep: fq_kv_quant time and HBM bandwidth vs number of head
vectors (L2 flushed before each timed launch; CUDA events on the launching stream)."""
import json
import sys

import torch

import paper_2410_09426_b200 as fq

dev = torch.device("cuda:0")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
res = []
for D in (128, 64):
    for R in (16384, 65536, 131072, 262144, 1048576, 4194304):
        kv = torch.randn((R, D), device=dev).half()
        ph = torch.linalg.qr(torch.randn((D, D), device=dev))[0].half()
        q = torch.empty((R, D // 2), dtype=torch.uint8, device=dev)
        s = torch.empty(R, device=dev)
        z = torch.empty(R, dtype=torch.int8, device=dev)
        for _ in range(3):
            fq.fq_kv_quant(kv, ph, 0.95, q, s, z)
        ts = []
        for _ in range(20):
            flush.zero_()
            torch.cuda._sleep(200_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fq.fq_kv_quant(kv, ph, 0.95, q, s, z)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        ms = ts[len(ts) // 2]
        by = R * (2 * D + D // 2 + 5)
        res.append({"D": D, "R": R, "us": round(ms * 1e3, 2), "gbs": round(by / ms / 1e6, 1)})
        print(json.dumps(res[-1]), flush=True)
json.dump(res, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/kv_sweep.json", "w"), indent=1)
