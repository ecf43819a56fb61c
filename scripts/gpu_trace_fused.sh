#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for s in "--N 6144 --K 4096" "--N 4096 --K 4096" "--N 28672 --K 4096"; do
  timeout 60 python scripts/trace_dec.py $s --flush --fused; timeout 60 python scripts/trace_dec.py $s --flush
done > gpurun_out/trace_fused.txt 2>&1
cat gpurun_out/trace_fused.txt | grep -v "TMA issue\|MMA issued"
