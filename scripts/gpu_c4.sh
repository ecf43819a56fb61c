#!/bin/bash
# C4 (decode) bench: fused decode linear vs the two-kernel path
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python bench.py --config C4 --steps 30 --warmup 5 --no-cpu --no-e2e --no-kv ${C4_ARGS} > gpurun_out/bench_C4_fused.json 2> gpurun_out/bench_C4_fused.err
timeout 300 python bench.py --config C4 --steps 30 --warmup 5 --no-cpu --no-e2e --no-kv --no-fp16 --no-fused > gpurun_out/bench_C4_unfused.json 2> gpurun_out/bench_C4_unfused.err
for f in fused unfused; do python - "$f" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/bench_C4_{sys.argv[1]}.json"))
print(sys.argv[1], d["ms_per_step"], d["value"], d["gpu_launches"], d["roofline"]["frac"], d.get("fp16_baseline"))
print({k: (v.get("linear_us"), v.get("tq_us"), v.get("gemm_us")) for k, v in d["kernels"].items()})
f6 = d["fig6_transform_overhead"]; print("int4-only", f6["int4_gemm_only_step_ms"], {k: v["marginal_us"] for k, v in f6["per_transform"].items()})
PY
done
tail -3 gpurun_out/bench_C4_fused.err
