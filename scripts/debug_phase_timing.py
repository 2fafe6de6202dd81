"""Debug: k_scan phase stamps (build with -DMARS_PHASE_TIMING first, see
scripts/gpu_phase_timing.sh).  Runs a few non-graph steps at 1M sessions,
flushing L2 before each, and prints the per-phase min/max stamps."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2604_26963_b200.engine import MarsEngine, make_config  # noqa: E402
from paper_2604_26963_b200.snapshot import snapshot_v1  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
variant = sys.argv[2] if len(sys.argv) > 2 else "headroom"
policy = sys.argv[3] if len(sys.argv) > 3 else "mars"
if variant == "headroom":
    snap = snapshot_v1(n, seed=0)
else:
    from tests._variants import reclaim_heavy
    snap = reclaim_heavy(n, 91, policy)
eng = MarsEngine(max_rows=snap.n, max_queue=max(len(snap.queue), 1),
                 config=make_config(initial_window=snap.initial_window, policy=policy))
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
eng.lib.mars_set_stream(eng.ctx, stream.cuda_stream)
eng.load_snapshot(snap)
if "s5" in sys.argv[4:]:  # the block-ID manager attached (the bench's default step)
    from paper_2604_26963_b200.kvstore import KvBlockManager
    kvm = KvBlockManager(eng, snap.total_blocks,
                         max_blocks_per_row=int(-(-(int(snap.cols["context"].max()) + 4096) // 16)))
    kvm.load_snapshot_tables(snap)
eng.checkpoint()
si = eng.step_in(snap.now, policy == 'mars', snap.active_tools, 0, snap.worker_slots)
eng.set_profiling(True)
for it in range(4):
    eng.restore()
    eng.flush_l2(512 << 20)
    print(f"--- step {it}", flush=True)
    eng.enqueue(si)
    eng.lib.mars_sync(eng.ctx)
    torch.cuda.synchronize()
    if it == 0:
        res = eng.fetch()
        print("diag", res.diag, "ret", len(res.ret_rows), "adm", len(res.admitted_rows),
              "exp", len(res.expired_rows), "ready", res.n_ready, "promoted", res.n_promoted,
              "dec", len(res.decode_rows), "pre", len(res.prefill_rows), flush=True)
    print({k: round(v * 1000, 1) for k, v in eng.kernel_times().items()}, flush=True)

# the same step captured in the CUDA graph (the bench's timed path): the stamp
# gaps between kernels are then the real inter-kernel gaps
eng.set_profiling(False)
eng.set_graph(True)
for it in range(3):
    eng.restore()
    eng.flush_l2(512 << 20)
    print(f"--- graph step {it}", flush=True)
    eng.enqueue(si)
    eng.lib.mars_sync(eng.ctx)
    torch.cuda.synchronize()

# and without the L2 flush: what the cold-cache (code + data) misses cost
for it in range(3):
    eng.restore()
    torch.cuda.synchronize()
    print(f"--- graph step, no flush {it}", flush=True)
    eng.enqueue(si)
    eng.lib.mars_sync(eng.ctx)
    torch.cuda.synchronize()
