"""Summarise an .ncu-rep: key metrics, stall breakdown, hottest source lines."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
d = dict(zip(h, r[2]))
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.sum.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "sm__cycles_elapsed.avg.per_second"]
for k in keys:
    print(f"  {k} = {d.get(k)}")
st = {k: v for k, v in d.items() if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")}


def f(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


tot = sum(f(v) for v in st.values()) or 1
print("  stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {f(v) / tot * 100:.1f}%"
                             for k, v in sorted(st.items(), key=lambda x: -f(x[1]))[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(src)))
hh = r[1]
i = hh.index("Warp Stall Sampling (All Samples)")
s = hh.index("Source")
rows = [x for x in r[2:] if len(x) > i]
tot = sum(int(x[i]) for x in rows) or 1
for x in sorted(rows, key=lambda x: -int(x[i]))[:ntop]:
    print(f"  {int(x[i]) / tot * 100:5.1f}%  {x[s][:110]}")
