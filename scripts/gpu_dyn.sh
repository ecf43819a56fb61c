#!/bin/bash
# transform dynamic tile schedule: parity + C3/C5 bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_dyn.log 2>&1; echo "exit $?" >> gpurun_out/pytest_dyn.log
tail -3 gpurun_out/pytest_dyn.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-kv --no-fp16 > gpurun_out/bench_dyn.json 2>/dev/null
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_dyn.json"))
f6 = d["fig6_transform_overhead"]
print("step", d["ms_per_step"], "tq_frac", d["tq_roofline"]["frac"], "in_step", d["tq_roofline"]["in_step"]["frac"],
      "int4", f6["int4_gemm_only_step_ms"], {k: v["marginal_us"] for k, v in f6["per_transform"].items()},
      {k: v["tq_us"] for k, v in d["kernels"].items()})
PY
