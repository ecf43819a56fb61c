cd /root/repo
mkdir -p gpurun_out
cp paper_2410_09426_b200/libflatquant.so /tmp/base.so
for L in base k256a k256b k128p; do
  if [ $L != base ]; then cp paper_2410_09426_b200/libflatquant_$L.so paper_2410_09426_b200/libflatquant.so; fi
  echo "== $L"
  timeout 300 python -m pytest tests -q -m gpu --timeout 240 -p no:cacheprovider -x -k "decode" 2>&1 | tail -1
  timeout 120 python scripts/dec_sweep.py --tag $L --flush clean --iters 20
  timeout 120 python scripts/dec_sweep.py --tag $L --flush rotate --iters 20
  cp /tmp/base.so paper_2410_09426_b200/libflatquant.so
done
timeout 300 python scripts/fig5_sweep.py
