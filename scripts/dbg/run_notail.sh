cp paper_2410_09426_b200/libflatquant.so /tmp/base.so
cp paper_2410_09426_b200/libflatquant_notail.so paper_2410_09426_b200/libflatquant.so
python scripts/dbg/dbg_sk2.py > gpurun_out/dbg_notail.txt 2>&1
cp /tmp/base.so paper_2410_09426_b200/libflatquant.so
