#!/bin/bash
# A/B of the decode GEMM's split-K tail (cluster barrier split around the dequant) on C4:
# default library vs FQ_LIB=paper_2410_09426_b200/libflatquant_tail.so, alternating.
cd "$(dirname "$0")/.."
NEW=$PWD/paper_2410_09426_b200/libflatquant_tail.so
FQ_LIB=$NEW timeout 600 python -m pytest tests -q -m gpu -x -k "dec or fused or C4" 2>&1 | tail -1
for i in 1 2 3; do
  for v in old new; do
    if [ $v = new ]; then export FQ_LIB=$NEW; else unset FQ_LIB; fi
    python bench.py --config C4 --no-cpu --no-e2e --no-kv --no-fp16 --no-fig6 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], {k: v.get('linear_us', v.get('gemm_us')) for k, v in d['kernels'].items()})"
  done
done
