#!/bin/bash
# BN = 240 pair tiles (FQ_PAIR_BN=240): GEMM parity, then the C2 / C3 steps against the default widths
cd "$(dirname "$0")/.."
FQ_PAIR_BN=240 timeout 600 python -m pytest tests -q -m gpu -x --timeout 200 -p no:cacheprovider -k "gemm_i32_bit_exact or dequant or chain or asym_linear or k_cap" 2>&1 | tail -2
python scripts/gemm_shapes.py 2>/dev/null | head -20
FQ_PAIR_BN=240 python scripts/gemm_shapes.py 2>/dev/null | head -20
for r in 1 2; do
  for B in 0 240; do
    for C in C2 C3; do
      FQ_PAIR_BN=$B timeout 300 python bench.py --config $C --steps 20 --warmup 5 --no-cpu --no-e2e --no-kv --no-fp16 --no-fig6 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('BN $B $C', d['ms_per_step'], {k: v['gemm_us'] for k, v in d['kernels'].items()})"
    done
  done
done
