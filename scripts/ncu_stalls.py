"""Aggregate warp-stall reasons (sampling) for one kernel of an ncu report.
usage: python scripts/ncu_stalls.py report.ncu-rep kernel_regex"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, vals = rows[0], rows[2]
items = []
for h, v in zip(hdr, vals):
    if "smsp__pcsamp_warps_issue_stalled_" in h and not h.endswith("not_issued"):
        try:
            items.append((float(v), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(x for x, _ in items) or 1
for v, h in sorted(items, reverse=True)[:14]:
    print(f"{100*v/tot:5.1f}%  {h}")
