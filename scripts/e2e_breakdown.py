"""Where the e2e step's time goes (1M sessions): column upload, step, fetch,
against one contiguous pinned copy of the same bytes."""
import statistics
import time

import torch

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
