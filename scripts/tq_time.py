"""Transform launch time (L2 flushed) for the n2 = 128 decompositions at T = 2048 and 32768."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_09426_b200 as fq  # noqa: E402

dev = torch.device("cuda:0")
flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)
tag = os.path.basename(os.environ.get("FQ_LIB", "default"))
for n1, n2 in ((64, 128), (112, 128), (64, 64)):
    for T in (2048, 32768):
        x = torch.randn((T, n1 * n2), device=dev).half()
        p1 = torch.linalg.qr(torch.randn(n1, n1, device=dev))[0].half().contiguous()
        p2 = torch.linalg.qr(torch.randn(n2, n2, device=dev))[0].half().contiguous()
        q = torch.empty((T, n1 * n2 // 2), dtype=torch.uint8, device=dev)
        s = torch.empty(T, device=dev)
        for _ in range(2):
            fq.fq_transform_quant(x, n1, n2, p1, p2, 0.9, q, s)
        tot = 0.0
        for _ in range(10):
            flush.zero_()
            flush.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fq.fq_transform_quant(x, n1, n2, p1, p2, 0.9, q, s)
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        us = tot / 10 * 1e3
        print(json.dumps({"lib": tag, "n1xn2": f"{n1}x{n2}", "T": T, "us": round(us, 1),
                          "gbs": round(T * (2 * n1 * n2 + n1 * n2 // 2 + 4) / (us * 1e-6) / 1e9, 1)}))
        del x, q, s
