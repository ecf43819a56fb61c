cd /root/repo
mkdir -p gpurun_out
for s in "--N 4096 --K 4096" "--N 28672 --K 4096" "--N 6144 --K 4096"; do
  timeout 60 python scripts/trace_dec.py $s
  timeout 60 python scripts/trace_dec.py $s --flush
done
