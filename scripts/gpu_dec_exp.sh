#!/bin/bash
# decode GEMM experiment builds: decode parity tests + C4 in-step kernel costs per variant
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for L in default ${VARIANTS}; do
  if [ "$L" = default ]; then unset FQ_LIB; else export FQ_LIB=$PWD/paper_2410_09426_b200/libflatquant_$L.so; fi
  echo "== $L"
  timeout 300 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "decode or chain_llama3_8b" 2>&1 | tail -1
  timeout 300 python scripts/step_prefix.py --config C4 --reps 40 2>&1 | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
print(' '.join(f\"{r['last']}:{r['delta_us']}\" for r in rows[1:]), 'total', rows[-1]['prefix_us'])"
done
