"""Summarise a phase-timing log (scripts/gpu_phase_timing.sh output): the
last block named argv[2] (default: the last flushed graph step), the kernel
stamps relative to the step head, and the S5 kernels' first start / last end."""
import sys

lines = open(sys.argv[1]).read().split("\n")
tag = sys.argv[2] if len(sys.argv) > 2 else "--- graph step 2"
i0 = max(i for i, l in enumerate(lines) if l.strip() == tag)
t0 = None
for l in lines[i0 + 1:]:
    if l.startswith("---"):
        break
    if l.startswith("t0 "):
        t0 = int(l.split()[1])
    elif l.startswith("kvt") and t0:
        _, k, a, b = l.split()
        print(f"kvt {k} ({['exp_push', 'apply_step'][int(k)] if int(k) < 2 else k}) "
              f"start {(int(a) - t0) / 1e3:.2f} end {(int(b) - t0) / 1e3:.2f}")
    elif l.startswith("stamp"):
        print(l)
