#!/bin/bash
# Round-2 re-entry baseline on a fresh box: full GPU suite, C3/C4 bench lines, decode timelines.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1; echo "exit $?" >> gpurun_out/pytest_full.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
timeout 300 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu --no-e2e --no-kv > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
FQ_DEC_CFG=0 timeout 300 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu --no-e2e --no-kv --no-fp16 > gpurun_out/bench_C4_cfg0.json 2> gpurun_out/bench_C4_cfg0.err
for s in "--N 6144 --K 4096" "--N 4096 --K 4096" "--N 28672 --K 4096" "--N 4096 --K 14336"; do timeout 60 python scripts/trace_dec.py $s --flush; done > gpurun_out/trace_dec.txt 2>&1
tail -n 5 gpurun_out/pytest_full.log
