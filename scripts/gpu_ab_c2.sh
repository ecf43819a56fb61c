#!/bin/bash
# A/B of the C2 / C3 steps between the product library and an experiment build ($VAR)
cd "$(dirname "$0")/.."
for r in 1 2 3; do
  for L in default $VAR; do
    if [ "$L" = default ]; then unset FQ_LIB; else export FQ_LIB=$PWD/paper_2410_09426_b200/libflatquant_$L.so; fi
    for C in C2 C3; do
      timeout 300 python bench.py --config $C --steps 20 --warmup 5 --no-cpu --no-e2e --no-kv --no-fp16 --no-fig6 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('$L $C', d['ms_per_step'], {k: v['gemm_us'] for k, v in d['kernels'].items()})"
    done
  done
done
