#!/bin/bash
# A/B the bench across alternative builds of the library: LIBS="pf6 pf8" bash scripts/ab_lib.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cp paper_2410_09426_b200/libflatquant.so /tmp/libflatquant_base.so
python scripts/peaks.py > gpurun_out/ab_base.txt 2>&1
for L in $LIBS; do
  cp paper_2410_09426_b200/libflatquant_$L.so paper_2410_09426_b200/libflatquant.so
  python scripts/peaks.py > gpurun_out/ab_$L.txt 2>&1
done
cp /tmp/libflatquant_base.so paper_2410_09426_b200/libflatquant.so
for f in gpurun_out/ab_*.txt; do echo "== $f"; cat $f; done
