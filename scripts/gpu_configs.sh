#!/bin/bash
# Bench every BASELINE config on one GPU (C3 is bench.py's default line; C2/C4/C5 are extra lines).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for C in ${CONFIGS:-C2 C4 C5}; do
  timeout 600 python bench.py --config $C --steps 20 --warmup 5 --no-cpu --no-e2e --no-kv > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err
  echo "bench $C exit $?" >> gpurun_out/bench_$C.err
done
tail -n 2 gpurun_out/bench_C*.err; cat gpurun_out/bench_C*.json
