"""Summarise the ncu captures of one GPU session into profiles/ (tracked):
  profiles/<tag>_launches.txt      per-kernel share of the ncu launch list of the bench command
  profiles/<tag>_<name>.txt        --set full summary + top source lines of each capture
  profiles/ncu_traffic.json        dram bytes (read + write) per launch of each captured kernel,
                                   read by bench.py for roofline.traffic
usage: python scripts/make_profiles.py <tag> [gpurun_out] [out_dir]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
prof = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "profiles")
os.makedirs(prof, exist_ok=True)


def run(*args):
    return subprocess.run([sys.executable, *args], capture_output=True, text=True).stdout


launches = os.path.join(src, "launches.csv")
if os.path.exists(launches):
    with open(os.path.join(prof, f"{tag}_launches.txt"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none: python bench.py --steps 2 --warmup 3 "
                "--no-cpu --no-e2e --no-fp16 --no-kv --no-fig6 (C3).  Cold-cache serialised launches: compare shares.\n")
        f.write(run(os.path.join(ROOT, "scripts", "launch_summary.py"), launches))
        f.write("\n## last 8 launches = one step (4 linears x transform+quant, W4A4 GEMM)\n")
        f.write(run(os.path.join(ROOT, "scripts", "launch_summary.py"), launches, "--last", "8"))

traffic_path = os.path.join(prof, "ncu_traffic.json")
traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
for fn in sorted(os.listdir(src)):
    if not fn.endswith(".ncu-rep") or not fn.startswith("prof_"):
        continue
    name = fn[len("prof_"):-len(".ncu-rep")]
    rep = os.path.join(src, fn)
    with open(os.path.join(prof, f"{tag}_{name}.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none --import-source on: scripts/prof_kernels.py ({name})\n")
        f.write(run(os.path.join(ROOT, "scripts", "ncu_summary.py"), rep, "15"))
        f.write("## top CUDA source lines (stall samples)\n")
        f.write(run(os.path.join(ROOT, "scripts", "ncu_lines.py"), rep, "25"))
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) >= 3:
        d = dict(zip(rows[0], rows[2]))
        u = dict(zip(rows[0], rows[1]))

        def val(k):
            v = float(d[k])
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[k], 1)
        traffic[name] = {"kernel": d.get("Kernel Name", "")[:80],
                         "dram_bytes": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                         "duration_us": float(d["gpu__time_duration.sum"]) * (1e-3 if u["gpu__time_duration.sum"] == "nsecond" else 1),
                         "capture": f"{tag}: {fn}"}
json.dump(traffic, open(traffic_path, "w"), indent=1)
print(json.dumps(traffic, indent=1))
