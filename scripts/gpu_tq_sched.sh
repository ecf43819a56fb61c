#!/bin/bash
# A/B of the transform's dynamic tile schedule: static first chunk FQ_TQ_CH0, claims in flight
# FQ_TQ_DEPTH -- transform alone (L2 flushed) and the C3 step.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in ${COMBOS:-"2 1" "2 2" "3 2" "4 2"}; do
  set -- $v
  echo "== ch0 $1 depth $2"
  FQ_TQ_CH0=$1 FQ_TQ_DEPTH=$2 python scripts/tq_time.py 2>&1 | grep '"T": 2048'
  FQ_TQ_CH0=$1 FQ_TQ_DEPTH=$2 python bench.py --config C3 --no-cpu --no-e2e --no-kv --no-fp16 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['ms_per_step'], d['tq_roofline']['frac'], d['tq_roofline'].get('in_step',{}).get('frac'), {k:v['tq_us'] for k,v in d['kernels'].items()})"
done
