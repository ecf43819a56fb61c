cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu --timeout 240 -p no:cacheprovider -x -k "decode or asym_linear or chain_llama3_8b" > gpurun_out/pytest_quick.log 2>&1; echo "exit $?" >> gpurun_out/pytest_quick.log
timeout 120 python scripts/dec_sweep.py --tag tmemw8 --flush clean --iters 30
timeout 120 python scripts/dec_sweep.py --tag tmemw8 --flush rotate --iters 30
for S in 1 2 3 4; do FQ_DEC_SPLIT=$S timeout 120 python scripts/dec_sweep.py --tag tmemw8s$S --flush clean --iters 30; done
for s in "--N 4096 --K 4096" "--N 28672 --K 4096"; do timeout 60 python scripts/trace_dec.py $s --flush; done
timeout 300 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu --no-e2e --no-kv > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
