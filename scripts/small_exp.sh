cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu --timeout 240 -p no:cacheprovider -k "tile_tails or chain_llama3_8b or transform_quant_vs_oracle" > gpurun_out/pytest_small.log 2>&1; echo "exit $?" >> gpurun_out/pytest_small.log
timeout 300 python bench.py --config C4 --steps 30 --warmup 5 --no-cpu --no-kv > gpurun_out/bench_C4s.json 2> gpurun_out/bench_C4s.err
FQ_TQ_SMALL=0 timeout 300 python bench.py --config C4 --steps 30 --warmup 5 --no-cpu --no-kv > gpurun_out/bench_C4l.json 2> gpurun_out/bench_C4l.err
