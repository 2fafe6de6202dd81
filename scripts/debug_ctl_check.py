import os, sys
sys.path.insert(0, os.getcwd())
os.environ["MARS_DEBUG_LAUNCH"] = "1"
from paper_2604_26963_b200.engine import MarsEngine, make_config
from paper_2604_26963_b200.snapshot import snapshot_v1
for n in (1_000_000, 16_000_000):
    snap = snapshot_v1(n, seed=7, pool="headroom")
    eng = MarsEngine(max_rows=snap.n, max_queue=max(len(snap.queue), 1),
                     config=make_config(initial_window=snap.initial_window))
    eng.load_snapshot(snap)
    si = eng.step_in(snap.now, True, snap.active_tools, snap.queued_tools, snap.worker_slots)
    r = eng.step(si)
    print(n, r.status, len(r.admitted_rows), r.limit, r.slots, r.diag["sort_path"], r.pack_mode)
    eng.close()
