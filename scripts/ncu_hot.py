"""Top SASS instructions by warp-stall samples for one kernel of an ncu report.

usage: python scripts/ncu_hot.py report.ncu-rep kernel_regex [topN]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern,
                      "--print-source=sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
recs = []
for r in rows[1:]:
    if len(r) <= iss or not r[iss].strip():
        continue
    try:
        recs.append((int(r[iss]), r[ia], r[isrc].strip()))
    except ValueError:
        pass
tot = sum(x[0] for x in recs) or 1
print(f"total stall samples {tot}")
for s, a, src in sorted(recs, reverse=True)[:top]:
    print(f"{100.0*s/tot:5.1f}%  {a[-5:]}  {src}")
