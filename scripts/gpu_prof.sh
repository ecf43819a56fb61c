#!/bin/bash
# ncu captures: launch list of a short bench run + full sets of the top kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-fp16 > gpurun_out/ncu_bench.log 2>&1
for LIN in ${PROF_LINEARS:-P_ug P_d}; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_tc05 -s 2 -c 1 -f \
    -o gpurun_out/prof_gemm_$LIN python scripts/prof_kernels.py --linear $LIN > gpurun_out/ncu_gemm_$LIN.log 2>&1
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:tq_ -s 2 -c 1 -f \
    -o gpurun_out/prof_tq_$LIN python scripts/prof_kernels.py --linear $LIN > gpurun_out/ncu_tq_$LIN.log 2>&1
done
ls -la gpurun_out
