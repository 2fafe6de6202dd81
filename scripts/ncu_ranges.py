"""Warp instructions and stall samples of one kernel bucketed by source-line
ranges (the --import-source copy of the file in the report).
usage: python scripts/ncu_ranges.py report.ncu-rep kernel_regex file.cu a-b[,c-d...]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep, kern, fn, spec = sys.argv[1:5]
ranges = [tuple(int(x) for x in r.split("-")) for r in spec.split(",")]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern,
                      "--print-source=cuda,sass"], capture_output=True, text=True).stdout
agg, smp = defaultdict(int), defaultdict(int)
fname, ii, si = "?", None, None
for row in csv.reader(io.StringIO(out)):
    if len(row) >= 2 and row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row and row[0] == "Line No":
        ii = row.index("Instructions Executed")
        si = row.index("Warp Stall Sampling (All Samples)")
        continue
    if ii is None or len(row) <= ii or not row[0].isdigit():
        continue
    try:
        v, s = int(row[ii]), int(row[si])
    except ValueError:
        continue
    key = "other"
    if fname == fn:
        for a, b in ranges:
            if a <= int(row[0]) <= b:
                key = f"{a}-{b}"
                break
        else:
            key = f"{fn}:rest"
    else:
        key = fname
    agg[key] += v
    smp[key] += s
tot, stot = sum(agg.values()) or 1, sum(smp.values()) or 1
print("total warp instructions", tot, "stall samples", stot)
for k in sorted(agg, key=lambda k: -agg[k]):
    print(f"{k:>28}: {100 * agg[k] / tot:5.1f}% inst  {100 * smp[k] / stot:5.1f}% stall")
