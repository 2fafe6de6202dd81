"""Is the full-table column upload asynchronous for the host?  Host return
times of one 65 MB pinned torch copy and of MarsEngine.upsert from pinned
columns (separately pinned vs views of one pinned buffer)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_26963_b200.engine import MarsEngine, make_config, step_columns  # noqa: E402
from paper_2604_26963_b200.snapshot import snapshot_v1  # noqa: E402

snap = snapshot_v1(1_000_000, seed=0, pool="headroom")
eng = MarsEngine(max_rows=snap.n, max_queue=len(snap.queue),
                 config=make_config(initial_window=snap.initial_window))
eng.load_snapshot(snap)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
eng.lib.mars_set_stream(eng.ctx, stream.cuda_stream)
cols = step_columns()
sep = {k: torch.from_numpy(snap.cols[k]).pin_memory().numpy() for k in cols}
nb = sum(v.nbytes for v in sep.values())
big = torch.empty(nb + 16 * len(cols), dtype=torch.uint8).pin_memory()
bn = big.numpy()
views, off = {}, 0
for k in cols:
    a = snap.cols[k]
    v = bn[off:off + a.nbytes].view(a.dtype)
    v[:] = a
    views[k] = v
    off += (a.nbytes + 15) // 16 * 16
flat = torch.empty(nb, dtype=torch.uint8).pin_memory()
dflat = torch.empty(nb, dtype=torch.uint8, device="cuda")
print("is_pinned", big.is_pinned(), flat.is_pinned())


def host(fn, n=6):
    r = []
    for i in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        r.append(((t1 - t0) * 1e3, (t2 - t0) * 1e3))
    r = r[1:]
    return "host return %.3f ms, done %.3f ms" % (np.median([x[0] for x in r]),
                                                  np.median([x[1] for x in r]))


print("torch flat copy      ", host(lambda: dflat.copy_(flat, non_blocking=True)))
print("upsert, sep pinned   ", host(lambda: eng.upsert(sep)))
print("upsert, one buffer   ", host(lambda: eng.upsert(views)))
for k in ("phase", "ready_since", "rank"):
    print("upsert one column", k, host(lambda: eng.upsert({k: sep[k]})))
