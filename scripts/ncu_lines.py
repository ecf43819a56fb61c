"""Top source lines (or SASS instructions) of an .ncu-rep by warp-stall samples, with the dominant
stall reasons of each (needs -lineinfo).
usage: python scripts/ncu_lines.py rep.ncu-rep [N] [--sass]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 25
sass = "--sass" in sys.argv
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass" if sass else "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Kernel Name"):
        continue
    if r[0] in ("Line No", "Address"):
        hdr = r
        continue
    if hdr is None:
        continue
    d = dict(zip(hdr, r))
    key = "Warp Stall Sampling (All Samples)"
    if not d.get(key, "").isdigit():
        continue
    stalls = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
    where = d.get("Address", "") if sass else f"{fname}:{r[0]}"
    src = d.get("Source", "")
    rows.append((int(d[key]), where, src, stalls))
tot = sum(x[0] for x in rows) or 1
for s, w, src, st in sorted(rows, key=lambda x: -x[0])[:ntop]:
    top = ", ".join(f"{k} {v / max(s, 1) * 100:.0f}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
    print(f"{s / tot * 100:5.1f}%  {w:>24}  {src.strip()[:90]:90}  [{top}]")
