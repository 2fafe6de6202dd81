"""Warp-stall samples aggregated per CUDA source line for one kernel.
usage: python scripts/ncu_lines.py report.ncu-rep kernel_regex [topN]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern,
                      "--print-source=cuda,sass"], capture_output=True, text=True).stdout
agg = defaultdict(int)
src = {}
fname = "?"
for row in csv.reader(io.StringIO(out)):
    if len(row) >= 2 and row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if len(row) < 5 or row[0] in ("Line No", "Function Name"):
        continue
    try:
        s = int(row[4])
    except ValueError:
        continue
    key = (fname, row[0])
    agg[key] += s
    if row[1].strip():
        src[key] = row[1].strip()
tot = sum(agg.values()) or 1
print("total samples", tot)
for key, s in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100*s/tot:5.1f}% {key[0]}:{key[1]:>5}  {src.get(key, '')[:90]}")
