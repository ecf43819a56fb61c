#!/bin/bash
# fused decode linear: parity tests, C4 chain, and the C4 bench step
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest_fused.log 2>&1; echo "exit $?" >> gpurun_out/pytest_fused.log
tail -n 30 gpurun_out/pytest_fused.log
timeout 600 python -m pytest tests -q -m gpu -x --timeout 240 -p no:cacheprovider -k "chain or decode or host_buffer or determinism" > gpurun_out/pytest_chain.log 2>&1; echo "exit $?" >> gpurun_out/pytest_chain.log
tail -n 5 gpurun_out/pytest_chain.log
