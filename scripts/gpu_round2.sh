#!/bin/bash
# Round-2 measurement session: smoke + GPU tests, bench lines for every config, ncu launch lists and
# --set full captures of the top kernels (summarised into profiles/ by scripts/make_profiles.py).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
if [ -z "$NO_TESTS" ]; then bash scripts/gpu_tests.sh > /dev/null 2>&1; fi
for CFG in ${CONFIGS:-C3 C2 C4 C5}; do
  EXTRA=""; if [ "$CFG" = C5 ]; then EXTRA="--no-cpu --no-e2e --no-kv"; fi
  timeout 900 python bench.py --config $CFG $EXTRA > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err
  echo "bench $CFG exit $?" >> gpurun_out/bench_$CFG.err
done
if [ -z "$NO_NCU" ]; then
  for CFG in C3 C4; do
    timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$CFG.csv \
      python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu --no-e2e --no-fp16 --no-kv --no-fig6 > gpurun_out/ncu_bench_$CFG.log 2>&1
  done
  cp gpurun_out/launches_C3.csv gpurun_out/launches.csv
  for LIN in P_a P_o P_ug P_d; do
    timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm -s 2 -c 1 -f \
      -o gpurun_out/prof_gemm_$LIN python scripts/prof_kernels.py --linear $LIN > gpurun_out/ncu_gemm_$LIN.log 2>&1
    timeout 600 $NCU --set full --clock-control none --import-source on -k regex:tq_ -s 2 -c 1 -f \
      -o gpurun_out/prof_tq_$LIN python scripts/prof_kernels.py --linear $LIN > gpurun_out/ncu_tq_$LIN.log 2>&1
  done
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_dec -s 2 -c 1 -f \
    -o gpurun_out/prof_dec_P_a python scripts/prof_kernels.py --config C4 --linear P_a > gpurun_out/ncu_dec.log 2>&1
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_dec -s 2 -c 1 -f \
    -o gpurun_out/prof_fused_P_a python scripts/prof_kernels.py --config C4 --linear P_a --fused > gpurun_out/ncu_fused.log 2>&1
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_dec -s 2 -c 1 -f \
    -o gpurun_out/prof_fused_P_ug python scripts/prof_kernels.py --config C4 --linear P_ug --fused > gpurun_out/ncu_fused_ug.log 2>&1
  mkdir -p gpurun_out/prof
  cp profiles/ncu_traffic.json gpurun_out/prof/ 2>/dev/null
  python scripts/make_profiles.py ${TAG:-r2a} gpurun_out gpurun_out/prof > gpurun_out/make_profiles.log 2>&1
  for CFG in C4; do python scripts/launch_summary.py gpurun_out/launches_$CFG.csv > gpurun_out/prof/${TAG:-r2a}_launches_$CFG.txt; done
  rm -f gpurun_out/*.ncu-rep gpurun_out/launches*.csv
fi
du -sh gpurun_out; ls gpurun_out
