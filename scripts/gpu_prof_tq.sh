#!/bin/bash
# ncu full captures of the transform kernel (and GEMM) for the linears in PROF_LINEARS + a launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
TAG=${TAG:-r1b}
for LIN in ${PROF_LINEARS:-P_ug P_d}; do
  timeout 300 $NCU --set full --clock-control none --import-source on -k regex:${KREGEX:-tq_} -s 2 -c 1 -f \
    -o gpurun_out/${TAG}_tq_$LIN python scripts/prof_kernels.py --linear $LIN > gpurun_out/${TAG}_ncu_tq_$LIN.log 2>&1
done
if [ -n "$LAUNCHES" ]; then
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-fp16 > gpurun_out/${TAG}_ncu_bench.log 2>&1
fi
ls gpurun_out
