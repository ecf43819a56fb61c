#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for TOOL in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $TOOL --print-limit 20 python scripts/sanitize_small.py > gpurun_out/sanitizer_$TOOL.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_$TOOL.txt
  tail -4 gpurun_out/sanitizer_$TOOL.txt
done
