"""Debug: sharded step captured as one CUDA graph vs eager."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2604_26963_b200.engine import MarsEngine, make_config
from paper_2604_26963_b200.dist import ShardedEngine
from paper_2604_26963_b200.snapshot import F_LONG, snapshot_v1
snap = snapshot_v1(30_000, seed=81, pool="headroom")
eng = MarsEngine(max_rows=snap.n, max_queue=2 * len(snap.queue),
                 config=make_config(initial_window=snap.initial_window))
eng.load_snapshot(snap)
sh = ShardedEngine(eng, world=1, rank=0)
q = snap.queue
sh.set_queue(q, snap.cols["req_blocks"][q], (snap.cols["flags"][q] & F_LONG) != 0, np.arange(len(q)))
si = eng.step_in(snap.now, True, snap.active_tools, 0, snap.worker_slots)
print("mode", si.mode)
eng.checkpoint()
r = sh.step(si)
print("eager", r.status, len(r.expired_rows), len(r.admitted_rows), len(r.window_rows), r.diag)
eng.restore()
r = sh.step(si)
print("eager2", r.status, len(r.expired_rows), len(r.admitted_rows), len(r.window_rows))
eng.restore()
sh.capture(si)
for i in range(2):
    eng.restore()
    sh.replay()
    r = eng.fetch()
    print("replay", i, r.status, len(r.expired_rows), len(r.admitted_rows), len(r.window_rows), r.diag)
