#!/bin/bash
# transform: persistent grid (default) vs MULTI (a few tiles per CTA, several CTAs per SM)
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -q -m gpu -x --timeout 200 -p no:cacheprovider -k "transform or chain or pdl" 2>&1 | tail -2
FQ_TQ_MULTI=2 timeout 600 python -m pytest tests -q -m gpu -x --timeout 200 -p no:cacheprovider -k "transform_quant_vs_oracle or tile_tails or chain_llama3_8b" 2>&1 | tail -2
for M in 0 2 4; do
  FQ_TQ_MULTI=$M timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-kv --no-fp16 > gpurun_out/bench_multi$M.json 2>/dev/null
  python - $M <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/bench_multi{sys.argv[1]}.json"))
f6 = d["fig6_transform_overhead"]
print("multi", sys.argv[1], "step", d["ms_per_step"], "tq_frac", d["tq_roofline"]["frac"], "in_step", d["tq_roofline"]["in_step"]["frac"],
      "int4", f6["int4_gemm_only_step_ms"], {k: v["marginal_us"] for k, v in f6["per_transform"].items()},
      {k: v["tq_us"] for k, v in d["kernels"].items()})
PY
done
