"""Where the e2e step's time goes (1M sessions): column upload, step, fetch,
against one contiguous pinned copy of the same bytes."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26963_b200.engine import MarsEngine, make_config, step_columns
from paper_2604_26963_b200.snapshot import snapshot_v1

snap = snapshot_v1(1_000_000, seed=0, pool="headroom")
eng = MarsEngine(max_rows=snap.n, max_queue=len(snap.queue),
                 config=make_config(initial_window=snap.initial_window))
eng.load_snapshot(snap)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
eng.lib.mars_set_stream(eng.ctx, stream.cuda_stream)
eng.set_graph(True)
si = eng.step_in(snap.now, True, snap.active_tools, snap.queued_tools, snap.worker_slots)
eng.checkpoint()
pinned = {k: torch.from_numpy(snap.cols[k]).pin_memory().numpy() for k in step_columns()}
nbytes = sum(v.nbytes for v in pinned.values())
flat = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
dflat = torch.empty(nbytes, dtype=torch.uint8, device="cuda")


def t(fn, n=10, flush=False):
    out = []
    for i in range(n + 1):
        eng.restore()
        if flush:
            eng.flush_l2(512 << 20)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        if i:
            out.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(out)


def full():
    eng.upsert(pinned)
    eng.enqueue(si)
    eng.fetch()


def step():
    eng.enqueue(si)
    eng.fetch()


def raw():
    dflat.copy_(flat, non_blocking=True)


print(f"bytes {nbytes}")
print(f"one pinned copy   {t(raw):.3f} ms")
print(f"upsert            {t(lambda: eng.upsert(pinned)):.3f} ms")
print(f"step+fetch        {t(step):.3f} ms")
print(f"enqueue only      {t(lambda: eng.enqueue(si)):.3f} ms")
print(f"upsert+step+fetch {t(full):.3f} ms")
print(f"  same, L2 flushed before each {t(full, flush=True):.3f} ms")
print(f"upsert, L2 flushed before each {t(lambda: eng.upsert(pinned), flush=True):.3f} ms")
print(f"one pinned copy, L2 flushed    {t(raw, flush=True):.3f} ms")

import ctypes as C

from paper_2604_26963_b200 import _native as N


def cfetch():
    eng.enqueue(si)
    o = N.MarsStepOut()
    eng.lib.mars_step_fetch(eng.ctx, C.byref(o))


print(f"step+C fetch      {t(cfetch):.3f} ms")
eng.enqueue(si)
o = N.MarsStepOut()
eng.lib.mars_step_fetch(eng.ctx, C.byref(o))
t0 = time.perf_counter()
for _ in range(20):
    r = eng.fetch.__wrapped__(eng) if hasattr(eng.fetch, "__wrapped__") else None
print("python wrapper cost measured via repeated fetch of the same outputs:")
t0 = time.perf_counter()
for _ in range(20):
    eng.fetch()
print(f"  fetch() x1      {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms")
t0 = time.perf_counter()
for _ in range(20):
    eng.fetch(copy=False)
print(f"  fetch(copy=False) x1 {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms")


# host-side return time of each piece (no synchronize inside): is the column
# upload asynchronous from the host's point of view?
def host_times(n=10):
    out = {"upsert": [], "enqueue": [], "fetch": [], "total": []}
    for i in range(n + 1):
        eng.restore()
        eng.flush_l2(512 << 20)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.upsert(pinned)
        t1 = time.perf_counter()
        eng.enqueue(si)
        t2 = time.perf_counter()
        eng.fetch()
        t3 = time.perf_counter()
        if i:
            out["upsert"].append((t1 - t0) * 1e3)
            out["enqueue"].append((t2 - t1) * 1e3)
            out["fetch"].append((t3 - t2) * 1e3)
            out["total"].append((t3 - t0) * 1e3)
    return {k: round(statistics.median(v), 3) for k, v in out.items()}


print("host return times (ms):", host_times())
# the same bytes as ONE pinned copy through the library's stream
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("13 column copies", lambda: eng.upsert(pinned)), ("one flat copy", raw)):
    ts = []
    for i in range(6):
        torch.cuda.synchronize()
        ev0.record(stream)
        fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        if i:
            ts.append(ev0.elapsed_time(ev1))
    print(f"device time {name}: {statistics.median(ts):.3f} ms")
