#!/bin/bash
# usage: KREGEX=... ARGS="--linear P_ug --gemm-impl 0" OUT=name bash scripts/gpu_prof_one.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s ${SKIP:-2} -c 1 -f \
  -o gpurun_out/${OUT} python scripts/prof_kernels.py ${ARGS} > gpurun_out/${OUT}.log 2>&1
echo "ncu exit $?" >> gpurun_out/${OUT}.log
