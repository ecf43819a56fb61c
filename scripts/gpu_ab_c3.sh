#!/bin/bash
# A/B of the C3 step between the product library and an experiment build ($VAR), 3 alternations;
# plus the wide transform tests and timing
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -q -m gpu -x --timeout 200 -p no:cacheprovider -k "wide or 128-224 or llama3_70b or transform_quant_vs_oracle" 2>&1 | tail -2
python scripts/wide_time.py
for r in 1 2 3; do
  for L in default $VAR; do
    if [ "$L" = default ]; then unset FQ_LIB; else export FQ_LIB=$PWD/paper_2410_09426_b200/libflatquant_$L.so; fi
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-kv --no-fp16 --no-fig6 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('$L', d['ms_per_step'])"
  done
done
unset FQ_LIB
