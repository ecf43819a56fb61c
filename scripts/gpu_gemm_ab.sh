#!/bin/bash
# GEMM A/B: bit-exact tests, then the bench with each GEMM implementation.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "gemm or w4a4" --timeout 120 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
for IMPL in ${IMPLS:-0 2}; do
  FQ_GEMM_IMPL=$IMPL timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --no-fp16 > gpurun_out/bench_impl$IMPL.json 2> gpurun_out/bench_impl$IMPL.err
done
