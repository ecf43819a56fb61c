#!/bin/bash
# Transform timing calibration + device timeline (instrumented build) on one B200.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python scripts/calib_tq.py > gpurun_out/calib.jsonl 2> gpurun_out/calib.err
for LIN in P_a P_d; do
  timeout 120 python scripts/trace_tq.py --linear $LIN > gpurun_out/trace_tq_$LIN.txt 2>&1
done
CFG=C4 timeout 300 python scripts/calib_tq.py > gpurun_out/calib_C4.jsonl 2>> gpurun_out/calib.err
cat gpurun_out/calib.jsonl; tail -5 gpurun_out/calib.err
