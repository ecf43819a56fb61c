"""INT8 dense tensor peak on this B200, the denominator of the W4A4 GEMM roofline (SURVEY.md
§8(d) "INT8 peak denominator"): (i) an own tcgen05.mma.kind::i8 issue loop on every SM
(instrumented build, csrc/fq_probe.cu: one elected thread per CTA / CTA pair issues back-to-back
M = 256 (pair) x N = 256 x K = 32 MMAs), (ii) cuBLASLt int8 through torch._int_mm on 8192^3.
Writes profiles/int8_peak.json; bench.py uses int8_tops from it."""
import ctypes
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FQ_TRACE_LIB"] = "1"
import paper_2410_09426_b200 as fq  # noqa: E402
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = fq.load()
out = (ctypes.c_ulonglong * 2)()
probe = {}
for pair, ts, n in ((1, 1, 256), (1, 0, 256), (0, 1, 256), (0, 0, 256), (1, 1, 192)):
    best = 0.0
    for _ in range(3):
        e = lib.fq_debug_mma_probe(pair | (ts << 1), n, 4000, 148, out)
        if e != 0:
            raise SystemExit(f"probe error {e}")
        ns, mmas = out[0], out[1]
        m = 256 if pair else 128
        units = 74 if pair else 148
        best = max(best, 2.0 * m * n * 32 * mmas * units / (ns * 1e-9) / 1e12)
    probe[f"{'pair' if pair else 'cta'}_M{256 if pair else 128}_N{n}_A{'tmem' if ts else 'smem'}"] = round(best, 1)

dev = torch.device("cuda:0")
a8 = torch.randint(-8, 8, (8192, 8192), device=dev, dtype=torch.int8)
b8 = torch.randint(-8, 8, (8192, 8192), device=dev, dtype=torch.int8).t()
for _ in range(5):
    torch._int_mm(a8, b8)
torch.cuda.synchronize()
best = 1e9
for _ in range(20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    torch._int_mm(a8, b8)
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
intmm = 2 * 8192 ** 3 / (best * 1e-3) / 1e12
clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader,nounits"],
                     capture_output=True, text=True).stdout.strip()
peak = max(probe.values())
res = {"int8_tops": peak, "probe_tops": probe, "cublaslt_int_mm_8192_tops": round(intmm, 1),
       "how": f"own tcgen05 kind::i8 issue loop, best shape ({max(probe, key=probe.get)}), 148 SMs; "
              f"cuBLASLt _int_mm 8192^3 {intmm:.0f} TOPS as the library cross-check",
       "gpu": torch.cuda.get_device_name(0), "sm_clocks_after": clk, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "int8_peak.json"), "w"), indent=1)
print(json.dumps(res))
