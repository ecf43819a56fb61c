#!/bin/bash
# C4: decode split choice with the cluster-residency count scaled by the measured co-residency
# (FQ_DEC_CLX=2) and two CTAs per SM allowed (FQ_DEC_GRIDCAP=2), against the default.
cd "$(dirname "$0")/.."
for i in 1 2; do
  for v in "1 1" "2 2" "1 2"; do
    set -- $v
    FQ_DEC_CLX=$1 FQ_DEC_GRIDCAP=$2 FQ_DEC_DEBUG=1 python bench.py --config C4 --no-cpu --no-e2e --no-kv --no-fp16 --no-fig6 2>gpurun_out/split_$1_$2.err | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('clx $1 cap $2', d['ms_per_step'], {k: v.get('linear_us') for k, v in d['kernels'].items()})"
    grep "decode GEMM" gpurun_out/split_$1_$2.err | sort | uniq | cut -c1-140
  done
done
