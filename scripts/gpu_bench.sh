#!/bin/bash
# Bench lines for the configs + INT8 peak probe on one B200 (outputs under gpurun_out/).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
python -c "import paper_2410_09426_b200.build as b; b.build(); b.build(trace=True)" > gpurun_out/build.log 2>&1
for CFG in ${CONFIGS:-C3 C4}; do
  timeout 600 python bench.py --config $CFG ${BENCH_ARGS} > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err
  echo "bench $CFG exit $?" >> gpurun_out/bench_$CFG.err
done
if [ -n "$INT8" ]; then timeout 300 python scripts/int8_peak.py > gpurun_out/int8_peak.log 2>&1; fi
for CFG in ${CONFIGS:-C3 C4}; do head -c 3000 gpurun_out/bench_$CFG.json; echo; tail -2 gpurun_out/bench_$CFG.err; done
tail -3 gpurun_out/int8_peak.log 2>/dev/null
