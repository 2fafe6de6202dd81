"""Warp instructions executed in a source-line range of one kernel (per file).
usage: python scripts/ncu_line_range.py report.ncu-rep kernel_regex file.cu first last"""
import csv, io, subprocess, sys
rep, kern, fname, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern,
                      "--print-source=cuda,sass"], capture_output=True, text=True).stdout
cur, ii, tot, rng = "?", None, 0, 0
for row in csv.reader(io.StringIO(out)):
    if len(row) >= 2 and row[0] == "File Path":
        cur = row[1].split("/")[-1]
        continue
    if row and row[0] == "Line No":
        ii = row.index("Instructions Executed")
        continue
    if ii is None or len(row) <= ii:
        continue
    try:
        n = int(row[ii])
    except ValueError:
        continue
    tot += n
    if cur == fname and row[0].strip().isdigit() and lo <= int(row[0]) <= hi:
        rng += n
print(f"total {tot}  range {rng}  ({100.0 * rng / max(tot, 1):.1f}%)")
