#!/bin/bash
# GPU test pass: smoke + pytest -m gpu (optionally a -k filter) on one B200.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -x ${PYTEST_K:+-k "$PYTEST_K"} ${PYTEST_FILES} > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/smoke.log; tail -n 30 gpurun_out/pytest_gpu.log
