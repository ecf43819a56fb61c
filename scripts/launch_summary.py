"""Summarise an ncu launch list (gpu__time_duration.sum per launch): per kernel name, the
count, mean/min duration and share of total time over the LAST `--steps` bench steps.
usage: python scripts/launch_summary.py launches.csv [--last N]"""
import collections
import csv
import re
import sys

path = sys.argv[1]
last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else None
rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
rows = [(int(r[0]), r[4], r[8], float(r[14])) for r in rows if r[12] == "gpu__time_duration.sum"]
OURS = ("g3::", "tq5::", "fq::", "tq_mma", "tq_simt", "gemm_pair", "gemm_tc05", "gemm_mma")
if last:
    rows = [r for r in rows if any(k in r[1] for k in OURS)][-last:]
agg = collections.OrderedDict()
for _, name, grid, ns in rows:
    short = re.sub(r"\(.*$", "", name.replace("void ", "")) + f" grid{grid}"
    a = agg.setdefault(short, [])
    a.append(ns)
tot = sum(ns for *_, ns in rows)
ours = sum(ns for _, n, _, ns in rows if any(k in n for k in OURS))
print(f"{len(rows)} launches, total {tot / 1e3:.1f} us, this library's kernels {ours / tot * 100:.1f}% of it")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v) / tot * 100:6.2f}%  n={len(v):3d}  mean {sum(v) / len(v) / 1e3:9.2f} us  min {min(v) / 1e3:9.2f} us  {k}")
