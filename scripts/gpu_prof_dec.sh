#!/bin/bash
# ncu captures of the decode GEMM (gate/up and o_proj shapes) and the wide transform, plus the
# launch list of the C4 (decode) bench step.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for SH in gate_up o_proj; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_dec -s 2 -c 1 -f \
    -o gpurun_out/prof_dec_$SH python scripts/dec_sweep.py --only $SH --iters 2 --flush clean > gpurun_out/ncu_dec_$SH.log 2>&1
done
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:tq_wide -s 2 -c 1 -f \
  -o gpurun_out/prof_tq_wide python scripts/prof_wide.py > gpurun_out/ncu_tq_wide.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C4.csv \
  python bench.py --config C4 --steps 2 --warmup 3 --no-cpu --no-e2e --no-fp16 --no-kv > gpurun_out/ncu_bench_C4.log 2>&1
ls -la gpurun_out
