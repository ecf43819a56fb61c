#!/bin/bash
# One GPU session: smoke + parity tests (+ optional bench), each step under its own timeout.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -p no:cacheprovider -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
if [ -n "$BENCH" ]; then
  timeout 600 python bench.py $BENCH > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
fi
tail -n 3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log
