#!/bin/bash
# Full GPU validation: smoke, every GPU test, bench lines for C3 (default) + C2/C4/C5, decomposition sweep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
CONFIGS="${CONFIGS:-C2 C4 C5}" bash scripts/gpu_configs.sh > /dev/null 2>&1
timeout 300 python scripts/fig5_sweep.py > gpurun_out/fig5.jsonl 2>&1
tail -n 2 gpurun_out/smoke.log gpurun_out/pytest_gpu.log
