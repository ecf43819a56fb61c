"""Top CUDA source lines of an .ncu-rep by warp-stall samples (needs -lineinfo).
usage: python scripts/ncu_lines.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname = [], "?"
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if len(r) > 5 and r[4].isdigit():
        rows.append((int(r[4]), fname, r[0], r[1]))
tot = sum(x[0] for x in rows) or 1
for s, f, ln, src in sorted(rows, reverse=True)[:ntop]:
    print(f"{s / tot * 100:5.1f}%  {f}:{ln}  {src.strip()[:110]}")
