cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 240 -p no:cacheprovider -k "gemm or w4a4 or asym_linear or chain" > gpurun_out/pytest_bn.log 2>&1; echo "exit $?" >> gpurun_out/pytest_bn.log
for BN in 256 192 160; do FQ_PAIR_BN=$BN timeout 120 python scripts/gemm_bn_sweep.py --tag bn$BN; done
timeout 120 python scripts/gemm_bn_sweep.py --tag auto
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-kv > gpurun_out/bench_C3bn.json 2> gpurun_out/bench_C3bn.err
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu --no-e2e --no-kv > gpurun_out/bench_C2bn.json 2> gpurun_out/bench_C2bn.err
FQ_TQ_IMPL=1 timeout 300 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu --no-e2e --no-kv > gpurun_out/bench_C4tq1.json 2> gpurun_out/bench_C4tq1.err
