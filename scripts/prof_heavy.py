"""One step of a heavy-reclaim 1M snapshot (for ncu captures of k_walk/k_scan)."""
import sys
sys.path.insert(0, ".")
from paper_2604_26963_b200.engine import MarsEngine, make_config  # noqa: E402
from tests._variants import reclaim_heavy  # noqa: E402

policy = sys.argv[1] if len(sys.argv) > 1 else "mars"
snap = reclaim_heavy(1_000_000, 91, policy)
eng = MarsEngine(max_rows=snap.n, max_queue=max(len(snap.queue), 1),
                 config=make_config(initial_window=snap.initial_window, policy=policy))
eng.load_snapshot(snap)
eng.checkpoint()
si = eng.step_in(snap.now, policy == "mars", snap.active_tools, 0, snap.worker_slots)
for _ in range(3):
    eng.restore()
    eng.flush_l2(512 << 20)
    r = eng.step(si)
print("evictions", len(r.evict_rows), r.diag)
