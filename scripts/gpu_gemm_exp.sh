#!/bin/bash
# GEMM experiment builds: throughput on the config shapes for each variant library.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OUT=gpurun_out/gemm_exp.jsonl; : > $OUT
timeout 300 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "gemm_i32_bit_exact or dequant or asym_linear" > gpurun_out/pytest_gemm.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gemm.log
IMPLS=${IMPLS:-0} timeout 300 python scripts/gemm_shapes.py >> $OUT 2>&1
for L in ${VARIANTS}; do
  FQ_LIB=$PWD/paper_2410_09426_b200/libflatquant_$L.so IMPLS=${IMPLS:-0} timeout 300 python scripts/gemm_shapes.py >> $OUT 2>&1
done
tail -2 gpurun_out/pytest_gemm.log; cat $OUT
