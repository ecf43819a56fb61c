#!/bin/bash
# One GPU session: smoke, GPU parity tests, bench, ncu launch list, ncu full captures.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
if [ -z "$NO_TESTS" ]; then
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
if [ -z "$NO_NCU" ]; then
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-fp16 > gpurun_out/ncu_bench.log 2>&1
for LIN in ${PROF_LINEARS:-P_a P_o P_ug P_d}; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm -s 2 -c 1 -f \
    -o gpurun_out/prof_gemm_$LIN python scripts/prof_kernels.py --linear $LIN > gpurun_out/ncu_gemm_$LIN.log 2>&1
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:tq_ -s 2 -c 1 -f \
    -o gpurun_out/prof_tq_$LIN python scripts/prof_kernels.py --linear $LIN > gpurun_out/ncu_tq_$LIN.log 2>&1
done
fi
ls -la gpurun_out
tail -n 3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json
