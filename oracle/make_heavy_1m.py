"""Freeze the CPU oracle's outputs for the heavy-reclaim / tick-gridded
snapshot steps at 1M sessions (tests/golden/heavy_1m.json).

At 1M sessions the oracle's reclaimer (one O(N log N) candidate sort per
failed claim, as the reference's scheduler.py:228-267 does) takes minutes per
step, too long to rerun inside the GPU test session, so its canonical
outputs (every decision plus the SHA-256 of each post-step column) are
frozen here.  The same oracle is pinned to the reference itself on these
variants at 30K sessions (tests/golden/heavy_steps.json, written by
oracle/make_golden.py --only heavy; checked by tests/test_oracle_golden.py).

Run:  python oracle/make_heavy_1m.py [--jobs 4]        TEST INFRASTRUCTURE ONLY.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from multiprocessing import get_context

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)

CASES_1M = [
    dict(n=1_000_000, seed=91, kind="reclaim_heavy", policy="mars", grid=False),
    dict(n=1_000_000, seed=92, kind="reclaim_heavy", policy="mars", grid=True),
    dict(n=1_000_000, seed=93, kind="reclaim_heavy", policy="fcfs", grid=True),
    dict(n=1_000_000, seed=94, kind="reclaim_heavy", policy="program_priority", grid=False),
    dict(n=1_000_000, seed=95, kind="reclaim_heavy", policy="static_ttl", grid=True),
    dict(n=1_000_000, seed=96, kind="reclaim_heavy", policy="dynamic_ttl", grid=False),
    dict(n=1_000_000, seed=97, kind="reclaim_heavy", policy="mars", grid=True,
         enable_coordinator=False),
]


def run(case):
    from oracle.make_golden import heavy_kw, heavy_snapshot
    from oracle.snapshot_step import run_step
    from tests._canon import canon, digest

    t0 = time.time()
    snap = heavy_snapshot(case)
    out = digest(canon(run_step(snap, **heavy_kw(case))))
    print(f"  {case}: {time.time() - t0:.0f}s evictions {len(out['evictions'])}", flush=True)
    return dict(case=case, out=out)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=4)
    a = ap.parse_args(argv)
    with get_context("fork").Pool(a.jobs) as pool:
        res = pool.map(run, CASES_1M)
    path = os.path.join(REPO, "tests", "golden", "heavy_1m.json")
    with open(path, "w") as fh:
        json.dump(res, fh, separators=(",", ":"))
    print("wrote", path)


if __name__ == "__main__":
    main()
