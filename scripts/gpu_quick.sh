#!/bin/bash
# Quick GPU iteration: selected parity tests (PYTEST_K) + a short bench, each under its own timeout.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout ${PYTEST_TIMEOUT:-600} python -m pytest tests -q -m gpu --timeout 240 -p no:cacheprovider -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_quick.log 2>&1; echo "exit $?" >> gpurun_out/pytest_quick.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench exit $?" >> gpurun_out/bench_quick.err
tail -n 15 gpurun_out/pytest_quick.log; cat gpurun_out/bench_quick.json; tail -3 gpurun_out/bench_quick.err
