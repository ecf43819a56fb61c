cd /root/repo
mkdir -p gpurun_out
for BN in 0 192 160 128 96 64; do
  if [ $BN = 0 ]; then timeout 120 python scripts/gemm_bn_sweep.py --tag auto; else FQ_PAIR_BN=$BN timeout 120 python scripts/gemm_bn_sweep.py --tag bn$BN; fi
done
for BN in 96 64; do FQ_PAIR_BN=$BN timeout 300 python -m pytest tests -q -m gpu --timeout 240 -p no:cacheprovider -k "gemm_i32_bit_exact and impl0" 2>&1 | tail -1; done
