"""Bit-exactness of the W4A4 GEMM (int32 accumulators) against the oracle on a few shapes with
tails, for whichever library FQ_LIB selects (experiment builds) and the pair-kernel widths."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2410_09426_b200 as fq  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
bad = 0
for impl in (0, 3, 4, 5, 7):
    for T, N, K in [(300, 520, 4096), (2048, 4096, 4096), (257, 200, 1056), (130, 264, 28672)]:
        qa = synth.random_codes(T, K, seed=T, tag="qa")
        qw = synth.random_codes(N, K, seed=N, tag="qw")
        fq.fq_set_gemm_impl(impl)
        acc = fq.w4a4_gemm_i32(torch.from_numpy(O.pack_int4(qa)).to(dev), torch.from_numpy(O.pack_int4(qw)).to(dev))
        torch.cuda.synchronize()
        ok = np.array_equal(acc.cpu().numpy().astype(np.int64), O.int_gemm(qa, qw))
        bad += not ok
        print(f"impl {impl} T={T} N={N} K={K}: {'ok' if ok else 'MISMATCH'}", flush=True)
fq.fq_set_gemm_impl(0)
print("ALL OK" if bad == 0 else f"{bad} MISMATCHES")
