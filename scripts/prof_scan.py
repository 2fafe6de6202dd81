"""One headroom step at N sessions (argv[1]; argv[2] == "s5": with S5) for ncu:
launch 1 warms up, launch 2 is the one to capture (ncu -k regex:k_scan -s 1 -c 1)."""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_2604_26963_b200.engine import MarsEngine, make_config  # noqa: E402
from paper_2604_26963_b200.snapshot import snapshot_v1  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16_000_000
snap = snapshot_v1(n, seed=7, pool="headroom")
eng = MarsEngine(max_rows=snap.n, max_queue=max(len(snap.queue), 1),
                 config=make_config(initial_window=snap.initial_window))
eng.load_snapshot(snap)
if len(sys.argv) > 2 and sys.argv[2] == "s5":  # the block-ID manager attached
    from paper_2604_26963_b200.kvstore import KvBlockManager
    kvm = KvBlockManager(eng, snap.total_blocks,
                         max_blocks_per_row=int(-(-(int(snap.cols["context"].max()) + 4096) // 16)))
    kvm.load_snapshot_tables(snap)
si = eng.step_in(snap.now, True, snap.active_tools, snap.queued_tools, snap.worker_slots)
eng.checkpoint()
for _ in range(2):
    eng.restore()
    eng.flush_l2(512 << 20)
    r = eng.step(si)
    assert r.status == 0, r.status
print("ok", n)
