#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -q -m gpu -x --timeout 300 -p no:cacheprovider -k "transform or chain or tails or weight_prep or schedule or p2_identity or abi_edges" 2>&1 | tail -2
python scripts/tq_time.py; FQ_LIB=$PWD/paper_2410_09426_b200/libflatquant_oldtq.so python scripts/tq_time.py
for L in default oldtq; do
  if [ "$L" = default ]; then unset FQ_LIB; else export FQ_LIB=$PWD/paper_2410_09426_b200/libflatquant_$L.so; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-kv --no-fp16 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); f=d['fig6_transform_overhead']; print('$L C3', d['ms_per_step'], {k: v['marginal_us'] for k, v in f['per_transform'].items()}, {k: v['tq_us'] for k, v in d['kernels'].items()})"
done
