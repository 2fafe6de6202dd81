"""Summarise ncu captures into profiles/ (tracked).

usage: python scripts/ncu_summary.py gpurun_out/prof.ncu-rep gpurun_out/launches.csv tag

Writes profiles/ncu_summary_<tag>.json (per-kernel duration, DRAM bytes,
throughput, occupancy, top stall reasons -- from the --set full capture) and
profiles/launches_<tag>.csv (the per-launch gpu__time_duration list of the
same bench command, with each kernel's share of the step).
"""

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
prof = os.path.join(root, "profiles")
os.makedirs(prof, exist_ok=True)

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "registers": "launch__registers_per_thread",
}
idx = {k: hdr.index(v) for k, v in want.items() if v in hdr}
name_i = hdr.index("Kernel Name")
stall_cols = [(i, h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for i, h in enumerate(hdr)
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
per = defaultdict(list)
for r in rows[2:]:
    name = r[name_i].split("(")[0]
    d = {}
    for k, i in idx.items():
        try:
            d[k] = float(r[i])
        except ValueError:
            d[k] = r[i]
    # normalise units: ncu reports bytes in the unit row (MB/KB/...)
    for k in ("dram_read_MB", "dram_write_MB"):
        u = units[idx[k]] if k in idx else ""
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
        d[k] = d.get(k, 0.0) * scale
    du = units[idx["duration_us"]]
    d["duration_us"] *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(du, 1.0)
    st = []
    for i, h in stall_cols:
        try:
            st.append((float(r[i]), h))
        except ValueError:
            pass
    tot = sum(v for v, _ in st) or 1.0
    d["top_stalls"] = [f"{h} {100 * v / tot:.0f}%" for v, h in sorted(st, reverse=True)[:4]]
    per[name].append(d)
summary = {}
for name, ds in per.items():
    d0 = dict(ds[-1])
    d0["captures"] = len(ds)
    d0["dram_bytes_per_launch"] = int((d0["dram_read_MB"] + d0["dram_write_MB"]) * 1e6)
    summary[name] = d0

# launch list: shares of the step
SETUP = ("k_flush", "k_scatter", "k_gather", "k_scatter_cols", "k_kv_bulk_scan", "k_kv_bulk_fill")
shares = defaultdict(float)
total = 0.0
if os.path.exists(launches):
    lines = [l for l in open(launches) if l.startswith('"')]
    lr = list(csv.reader(io.StringIO("".join(lines))))
    h = lr[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    with open(os.path.join(prof, f"launches_{tag}.csv"), "w") as fh:
        fh.write("kernel,duration_ns\n")
        for r in lr[1:]:
            if r[mi] != "gpu__time_duration.sum":
                continue
            k = r[ki].split("(")[0]
            v = float(r[vi].replace(",", ""))
            fh.write(f"{k},{v}\n")
            # one-time setup (the block tables' bulk fill, the snapshot's
            # column scatter) and the L2 flush are not part of a step
            if k.startswith("k_") and k not in SETUP:
                shares[k] += v
                total += v
summary["_step_share_cold_serialised"] = {k: round(v / total, 4) for k, v in
                                          sorted(shares.items(), key=lambda x: -x[1])} if total else {}
with open(os.path.join(prof, f"ncu_summary_{tag}.json"), "w") as fh:
    json.dump(summary, fh, indent=1)
print(json.dumps({k: (v.get("duration_us"), v.get("dram_bytes_per_launch"))
                  for k, v in summary.items() if not k.startswith("_")}, indent=1))
print(summary["_step_share_cold_serialised"])
