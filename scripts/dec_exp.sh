cd /root/repo
mkdir -p gpurun_out
for F in write clean rotate; do
  timeout 120 python scripts/dec_sweep.py --tag base --flush $F --iters 20
  FQ_GEMM_IMPL=5 timeout 120 python scripts/dec_sweep.py --tag pair128 --flush $F --iters 20
done
for S in 1 2 4 8; do FQ_DEC_SPLIT=$S timeout 120 python scripts/dec_sweep.py --tag base --flush rotate --iters 20; done
cp paper_2410_09426_b200/libflatquant.so /tmp/base.so
for L in s3p3 one; do
  cp paper_2410_09426_b200/libflatquant_$L.so paper_2410_09426_b200/libflatquant.so
  for S in 0 2 4; do FQ_DEC_SPLIT=$S timeout 120 python scripts/dec_sweep.py --tag $L --flush rotate --iters 20; done
  cp /tmp/base.so paper_2410_09426_b200/libflatquant.so
done
