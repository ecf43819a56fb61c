#!/bin/bash
# decode: the four-GEMM chain (fused_probe gemm_only) and dec_shapes for the product library and $VARIANTS
cd "$(dirname "$0")/.."
for L in default $VARIANTS; do
  if [ "$L" = default ]; then unset FQ_LIB; else export FQ_LIB=$PWD/paper_2410_09426_b200/libflatquant_$L.so; fi
  python scripts/fused_probe.py --reps 20 | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('$L', {k: v for k, v in d.items() if 'gemm_only' in k})"
done
