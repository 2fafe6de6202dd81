"""Instructions executed (warp-level) per CUDA source line for one kernel.
usage: python scripts/ncu_insts.py report.ncu-rep kernel_regex [topN]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern,
                      "--print-source=cuda,sass"], capture_output=True, text=True).stdout
agg, smp, src = defaultdict(int), defaultdict(int), {}
fname = "?"
ii = si = None
for row in csv.reader(io.StringIO(out)):
    if len(row) >= 2 and row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row and row[0] == "Line No":
        ii = row.index("Instructions Executed")
        si = row.index("Warp Stall Sampling (All Samples)")
        continue
    if ii is None or len(row) <= ii:
        continue
    try:
        v = int(row[ii]); s = int(row[si])
    except ValueError:
        continue
    if not row[0].isdigit():
        continue
    key = (fname, int(row[0]))
    agg[key] += v
    smp[key] += s
    if row[1].strip():
        src[key] = row[1].strip()
tot = sum(agg.values()) or 1
stot = sum(smp.values()) or 1
print("total warp instructions", tot, "samples", stot)
for key, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100*v/tot:5.1f}% inst {100*smp[key]/stot:5.1f}% stall {key[0]}:{key[1]:>5}  {src.get(key, '')[:80]}")
