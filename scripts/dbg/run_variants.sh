cp paper_2410_09426_b200/libflatquant.so /tmp/base.so
for V in $VARIANTS; do
  cp paper_2410_09426_b200/libflatquant_$V.so paper_2410_09426_b200/libflatquant.so
  python scripts/dbg/dbg_sk2.py 2>&1 | grep -c "^tile" > gpurun_out/dbg_$V.txt
  python scripts/dbg/dbg_sk2.py 2>&1 | head -4 >> gpurun_out/dbg_$V.txt
done
cp /tmp/base.so paper_2410_09426_b200/libflatquant.so
