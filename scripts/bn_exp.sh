cd /root/repo
mkdir -p gpurun_out
timeout 120 python scripts/gemm_bn_sweep.py --tag base
cp paper_2410_09426_b200/libflatquant.so /tmp/base.so
cp paper_2410_09426_b200/libflatquant_a16.so paper_2410_09426_b200/libflatquant.so
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 240 -p no:cacheprovider -x -k "gemm_i32" 2>&1 | tail -1
timeout 120 python scripts/gemm_bn_sweep.py --tag a16
cp /tmp/base.so paper_2410_09426_b200/libflatquant.so
