"""Replays bench.py's call sequence with an error check after every call."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2604_26963_b200 import _native as N
from paper_2604_26963_b200.engine import MarsEngine, make_config
from paper_2604_26963_b200.snapshot import snapshot_v1

snap = snapshot_v1(200_000, seed=0)
eng = MarsEngine(max_rows=snap.n, max_queue=len(snap.queue), config=make_config(initial_window=snap.initial_window))
def chk(tag):
    rc = eng.lib.mars_sync(eng.ctx)
    print(tag, "ok" if rc == 0 else eng.lib.mars_last_error(eng.ctx).decode(), flush=True)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
eng.lib.mars_set_stream(eng.ctx, stream.cuda_stream); chk("set_stream")
eng.set_graph(True); chk("set_graph")
eng.load_snapshot(snap); chk("load")
eng.checkpoint(); chk("ckpt")
si = eng.step_in(snap.now, True, snap.active_tools, 0, snap.worker_slots)
eng.enqueue(si); chk("enqueue1")
r = eng.fetch(); chk("fetch1")
eng.restore(); chk("restore")
eng.enqueue(si); chk("enqueue2")
eng.restore(); chk("restore2")
eng.set_profiling(True); chk("prof")
eng.flush_l2(256 << 20); chk("flush")
eng.enqueue(si); chk("enqueue-prof")
print(eng.kernel_times()); chk("ktimes")
eng.set_graph(False); eng.restore(); eng.enqueue(si); chk("nograph-prof")
print(eng.kernel_times())
