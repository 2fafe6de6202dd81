"""Benchmark: one MARS scheduling step over a 1M-session table per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--sessions S] [--impl reference]

A *step* is one full pass of the hot path over the device-resident session
table (snapshot_v1, mix A, headroom pool): pin expiry, telemetry probe,
control-plane admission (refresh_pressure, pack_queue, AIMD window, admit),
MLFQ aging, window top-128, the build_plan walk with chunk fitting and
reclamation, and S2 retention for the boundary rows.  Every timed step starts
from the same snapshot (device-side restore, untimed) with L2 flushed, so each
step repeats the identical decisions.

Multi-GPU (torchrun): ONE global 1M-session snapshot,
rows sharded rank mod N over data-parallel engine replicas (strong scaling);
global admission exchanges the probe counters (NCCL all-reduce) and the
admission entries (all-gather); time = max over ranks, value = the global
table's sessions per second.

``--impl reference`` times the reference CPU path (the oracle port of
agentsched, single-threaded CPython) on the same workload and prints the same
JSON line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sched steps/s & sessions/s at 1M sessions; KV evict/restore GB/s"
FALLBACK_HBM_GBS = 6650.0


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", FALLBACK_HBM_GBS)), "measured"
    return FALLBACK_HBM_GBS, "fallback"


def _ncu_traffic():
    """k_scan's DRAM bytes per launch (dram__bytes_read + write) from the
    newest committed ncu capture of this bench command (profiles/, written by
    scripts/ncu_summary.py; ncu cannot run inside the timed process)."""
    import glob
    caps = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_summary_r*.json")))
    if not caps:
        return None, None
    try:
        with open(caps[-1]) as fh:
            d = json.load(fh)
        return d.get("k_scan", {}).get("dram_bytes_per_launch"), os.path.basename(caps[-1])
    except Exception:
        return None, None


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def scan_bytes(snap) -> int:
    """Algorithmic bytes of one k_scan launch: phase+flags for
    every row; level, promos, wait_since, ready_since, kv for ready rows; the
    promotion write-back; deadline/pinned_blocks/plevel for pinned rows;
    req_blocks for queued rows; the expiry write-back + expired list."""
    import numpy as np

    from paper_2604_26963_b200.snapshot import DECODE, F_PINNED, F_QUEUED, PREFILL

    c = snap.cols
    ready = (c["phase"] == DECODE) | (c["phase"] == PREFILL)
    pinned = (c["flags"] & F_PINNED) != 0
    queued = (c["flags"] & F_QUEUED) != 0
    now = snap.now
    promo = ready & (c["level"] > 0) & (c["promos"] < 3) & (now - c["wait_since"] >= 10.0)
    expired = pinned & (c["deadline"] < now)
    return int(2 * snap.n + 22 * ready.sum() + 10 * promo.sum() + 13 * pinned.sum()
               + 4 * queued.sum() + 17 * expired.sum())


def step_bytes(snap) -> int:
    """Whole-step algorithmic bytes, SURVEY.md §8(d) accounting."""
    from paper_2604_26963_b200.snapshot import DECODE, F_BOUNDARY, F_PINNED, F_QUEUED, PREFILL

    c = snap.cols
    ready = (c["phase"] == DECODE) | (c["phase"] == PREFILL)
    now = snap.now
    promo = ready & (c["level"] > 0) & (c["promos"] < 3) & (now - c["wait_since"] >= 10.0)
    return int(snap.n * 1 + ready.sum() * 18 + promo.sum() * 10
               + ((c["flags"] & F_PINNED) != 0).sum() * 8
               + ((c["flags"] & F_BOUNDARY) != 0).sum() * 17
               + ((c["flags"] & F_QUEUED) != 0).sum() * 13)


def kv_sweep(device: int, batches=(1, 16, 256, 2048), reps: int = 3) -> dict:
    """BASELINE configs[3]: paged KV evict (HBM -> pinned host) / restore sweep,
    Llama-3-8B geometry (2 MiB per 16-token block, 32 layer-major pieces),
    scattered random block IDs, each call timed end to end through the ABI,
    against the measured pinned-copy peak of the host link."""
    import numpy as np

    from paper_2604_26963_b200.engine import MarsEngine
    from paper_2604_26963_b200.kvstore import (LLAMA3_8B_BLOCK_BYTES, LLAMA3_8B_LAYERS,
                                               KvBlockManager, host_link_peak)

    eng = MarsEngine(max_rows=64, max_queue=1, device=device)
    d2h, h2d, bidir = host_link_peak(eng, 1 << 30, 5)
    total, host_blocks = 8192, max(batches)
    kv = KvBlockManager(eng, total, max_blocks_per_row=16, block_bytes=LLAMA3_8B_BLOCK_BYTES,
                        layers=LLAMA3_8B_LAYERS, host_blocks=host_blocks)
    rng = np.random.default_rng(3)
    names = {0: "copy_engine_per_piece", 1: "sm_zero_copy", 2: "staged_dma"}
    sweep = []
    for n in batches:
        ids = rng.choice(total, size=n, replace=False).astype(np.uint32)
        for m in (0, 1, 2):
            for direction in ("evict", "restore"):
                fn = kv.evict if direction == "evict" else kv.restore
                fn(ids, 0, m)  # warm
                ts = []
                for _ in range(reps):
                    t0 = time.perf_counter()
                    fn(ids, 0, m)
                    ts.append(time.perf_counter() - t0)
                gbs = n * LLAMA3_8B_BLOCK_BYTES / min(ts) / 1e9
                sweep.append({"blocks": n, "method": names[m], "op": direction, "gbs": gbs})
    eng.close()
    big = [s for s in sweep if s["blocks"] == max(batches)]
    ev = max((s for s in big if s["op"] == "evict"), key=lambda s: s["gbs"])
    rs = max((s for s in big if s["op"] == "restore"), key=lambda s: s["gbs"])
    return {"evict_gbs": ev["gbs"], "evict_method": ev["method"], "restore_gbs": rs["gbs"],
            "restore_method": rs["method"], "peak_d2h_gbs": d2h, "peak_h2d_gbs": h2d,
            "peak_bidir_gbs": bidir, "evict_frac": ev["gbs"] / d2h, "restore_frac": rs["gbs"] / h2d,
            "block_bytes": LLAMA3_8B_BLOCK_BYTES, "batch_blocks": max(batches),
            "peak_source": "pinned cudaMemcpyAsync 1 GiB, best of 5, measured in this run",
            "sweep": sweep}


def kv_tier_run(block_bytes: int = 16384, key: str = "openhands_heavy40/mars") -> dict:
    """SURVEY.md §8(d) config (5), the KV path: the OpenHands-style heavy
    trace run whole on the device (devsim, event log byte-identical to the
    reference's) with the host tier following its decisions -- pins copied
    to pinned host memory, warm resumes copied back, running-session
    evictions and unpinned boundaries copied out -- at `block_bytes` per
    16-token block (the Llama-3-8B 2 MiB block would need 340 GB of HBM for
    this pool).  GB/s = bytes / time of the copy calls (synchronous, staged
    DMA), against the pinned-copy peak of the link measured here."""
    from paper_2604_26963_b200.devsim import EventLog, load_trace, run_device_simulation
    from paper_2604_26963_b200.engine import MarsEngine
    from paper_2604_26963_b200.kvstore import host_link_peak

    ref_dir = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(ref_dir, "sim_logs.json")) as fh:
        spec = json.load(fh)[key]
    traces = load_trace(os.path.join(ref_dir, spec["trace"]))
    total = spec["engine"]["total_blocks"]
    log, kv = EventLog(), {}
    tier = {"block_bytes": block_bytes, "host_blocks": 2 * total}
    t0 = time.perf_counter()
    run_device_simulation(traces, total, spec["engine"]["tool_worker_slots"], log=log,
                          kv_state=kv, kv_tier=tier)
    wall = time.perf_counter() - t0
    import hashlib
    same = hashlib.sha256(log.jsonl_bytes()).hexdigest() == spec["sha256"]
    eng = MarsEngine(max_rows=64, max_queue=1)
    d2h, h2d, _ = host_link_peak(eng, 1 << 30, 5)
    eng.close()
    out = {k: tier[k] for k in ("evict_blocks", "pin_blocks", "restore_blocks", "d2h_bytes",
                                "h2d_bytes", "d2h_s", "h2d_s", "d2h_gbs", "h2d_gbs")}
    out.update(trace=key, block_bytes=block_bytes, log_identical=same, run_wall_s=wall,
               peak_d2h_gbs=d2h, peak_h2d_gbs=h2d,
               d2h_frac=(tier["d2h_gbs"] or 0) / d2h, h2d_frac=(tier["h2d_gbs"] or 0) / h2d)
    return out


def hbm_sweep(device: int, sizes, steps: int = 5, warmup: int = 3, flush_mb: int = 512) -> list:
    """the step and its scan kernel on tables far beyond the
    126 MB L2 (L2 flushed before every step), where the 1M-session step's
    latency floor no longer hides the bandwidth the kernels reach."""
    import statistics as st

    import torch

    from paper_2604_26963_b200.engine import MarsEngine, make_config
    from paper_2604_26963_b200.snapshot import snapshot_v1

    peak, _ = _peaks()
    out = []
    for n in sizes:
        snap = snapshot_v1(n, seed=7, pool="headroom")
        eng = MarsEngine(max_rows=snap.n, max_queue=max(len(snap.queue), 1), device=device,
                         config=make_config(initial_window=snap.initial_window))
        eng.load_snapshot(snap)
        si = eng.step_in(snap.now, True, snap.active_tools, snap.queued_tools, snap.worker_slots)
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        eng.lib.mars_set_stream(eng.ctx, stream.cuda_stream)
        eng.checkpoint()
        eng.set_graph(True)
        for _ in range(warmup):
            eng.restore()
            eng.enqueue(si)
        torch.cuda.synchronize()
        ms = []
        for _ in range(steps):
            eng.restore()
            eng.flush_l2(flush_mb << 20)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            eng.enqueue(si)
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        eng.set_graph(False)
        eng.set_profiling(True)
        kt = []
        for _ in range(steps):
            eng.restore()
            eng.flush_l2(flush_mb << 20)
            eng.enqueue(si)
            kt.append(eng.kernel_times())
        eng.set_profiling(False)
        res = eng.fetch()
        scan_ms = st.median(k["k_scan"] for k in kt)
        sb = scan_bytes(snap)
        sbs = step_bytes(snap)
        step_ms = st.median(ms)
        out.append({"sessions": n, "status": int(res.status), "ms_per_step": step_ms,
                    "sessions_per_s": n / (step_ms * 1e-3),
                    "k_scan_ms": scan_ms, "k_scan_gbs": sb / (scan_ms * 1e-3) / 1e9,
                    "k_scan_frac": sb / (scan_ms * 1e-3) / 1e9 / peak,
                    "k_control_ms": st.median(k["k_control"] for k in kt),
                    "k_walk_ms": st.median(k["k_walk"] for k in kt),
                    "step_frac": sbs / (step_ms * 1e-3) / 1e9 / peak,
                    "table_mb": sum(v.nbytes for v in snap.cols.values()) / 1e6})
        eng.close()
        del snap
        torch.cuda.synchronize()
    return out


def regime_sweep(device: int, n: int, steps: int = 10, warmup: int = 3, flush_mb: int = 512) -> list:
    """The step on the regimes beyond the headroom snapshot, at 1M sessions
    (SURVEY.md §8(d) pressure pool; VERDICT r1 task 1): heavy reclamation
    (every running session holds 1-2 blocks, no free block: dozens of victims
    per step) under MARS and a comparison policy, and tick-gridded ties
    (every time on the 0.064 s grid, a batch admitted at `now`).  Same timing
    as the headline (graph launch, L2 flushed, state restored, CUDA events)."""
    import statistics as st

    import torch

    from paper_2604_26963_b200.engine import MarsEngine, make_config
    from paper_2604_26963_b200.snapshot import snapshot_v1
    from tests._variants import reclaim_heavy, tick_grid

    cases = [("reclaim_heavy", "mars", lambda: reclaim_heavy(n, 91, "mars")),
             ("reclaim_heavy_grid", "mars", lambda: tick_grid(reclaim_heavy(n, 92, "mars"), 92)),
             ("reclaim_heavy_grid", "fcfs", lambda: tick_grid(reclaim_heavy(n, 93, "fcfs"), 93)),
             ("reclaim_heavy", "program_priority", lambda: reclaim_heavy(n, 94, "program_priority")),
             ("tick_grid_headroom", "mars", lambda: tick_grid(snapshot_v1(n, seed=111), 111))]
    out = []
    for name, policy, mk in cases:
        snap = mk()
        due = policy == "mars"
        eng = MarsEngine(max_rows=snap.n, max_queue=max(len(snap.queue), 1), device=device,
                         config=make_config(initial_window=snap.initial_window, policy=policy))
        eng.load_snapshot(snap)
        si = eng.step_in(snap.now, due, snap.active_tools, snap.queued_tools, snap.worker_slots)
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        eng.lib.mars_set_stream(eng.ctx, stream.cuda_stream)
        eng.checkpoint()
        res = eng.step(si)
        eng.restore()
        eng.set_graph(True)
        for _ in range(warmup):
            eng.restore()
            eng.enqueue(si)
        torch.cuda.synchronize()
        ms = []
        for _ in range(steps):
            eng.restore()
            eng.flush_l2(flush_mb << 20)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            eng.enqueue(si)
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        eng.set_graph(False)
        eng.set_profiling(True)
        kt = []
        for _ in range(steps):
            eng.restore()
            eng.flush_l2(flush_mb << 20)
            eng.enqueue(si)
            kt.append(eng.kernel_times())
        eng.set_profiling(False)
        step_ms = st.median(ms)
        out.append({"regime": name, "policy": policy, "sessions": n, "status": int(res.status),
                    "ms_per_step": step_ms, "sessions_per_s": n / (step_ms * 1e-3),
                    "evictions": int(len(res.evict_rows)), "tokens": int(res.total_tokens),
                    "n_fullscan": res.diag["n_fullscan"], "ref_flags": res.diag["ref_flags"],
                    "ref_rounds": res.diag["ref_rounds"],
                    "k_scan_ms": st.median(k["k_scan"] for k in kt),
                    "k_walk_ms": st.median(k["k_walk"] for k in kt),
                    "k_control_ms": st.median(k["k_control"] for k in kt) if due else None})
        eng.close()
        del snap
        torch.cuda.synchronize()
    return out


def dropin_sweep(keys=("demo64/mars", "faceoff200/mars", "openhands_heavy40/mars")) -> list:
    """SURVEY.md §8(d) configs (1) and (5), the full loop: the reference's own
    ``agentsched.sim.run_simulation`` (baseline/_ref) on a frozen reference
    trace, once with the reference MarsPolicy and once with the INTEGRATION.md
    binding (GpuMarsPolicy + the B200 balance_and_admit).  Wall time of the
    whole run on the host clock, scheduling steps (plan_tick calls) per second
    for both arms, and whether the drop-in's event log is byte-identical to
    the reference's (the frozen SHA-256)."""
    import hashlib

    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref_dir) and ref_dir not in sys.path:
        sys.path.insert(1, ref_dir)
    try:
        from agentsched import baselines, control, sim, workload
    except ImportError:
        return [{"error": "agentsched (baseline/_ref) not importable"}]
    with open(os.path.join(ROOT, "tests", "golden", "sim_logs.json")) as fh:
        SIM = json.load(fh)

    from paper_2604_26963_b200.admission import balance_and_admit as gpu_bna
    from paper_2604_26963_b200.policy import GpuMarsPolicy

    out = []
    for key in keys:
        spec = SIM[key]
        traces = workload.load_trace(os.path.join(ROOT, "tests", "golden", spec["trace"]))
        params = sim.EngineParams(**spec["engine"])
        run = dict(spec["run"])
        if "controller" in run:
            run["controller"] = control.ControllerConfig(**run["controller"])
        row = {"trace": key, "sessions": len(traces)}
        for arm in ("reference", "b200"):
            pol = baselines.make_policy("mars") if arm == "reference" else GpuMarsPolicy()
            if arm == "b200":
                pol._engine()  # the device context: one-time setup, outside the timing
            ticks = [0]
            inner = pol.plan_tick

            def counted(*a, _inner=inner, _t=ticks, **k):
                _t[0] += 1
                return _inner(*a, **k)

            pol.plan_tick = counted
            orig = sim.balance_and_admit
            if arm == "b200":
                sim.balance_and_admit = gpu_bna
            try:
                t0 = time.perf_counter()
                res = sim.run_simulation(traces, params, pol, **run)
                dt = time.perf_counter() - t0
            finally:
                sim.balance_and_admit = orig
                if arm == "b200":
                    pol.close()
            data = b"".join(json.dumps(r, separators=(",", ":")).encode() + b"\n"
                            for r in res.events)
            row[arm] = {"wall_s": dt, "steps": ticks[0], "steps_per_s": ticks[0] / dt,
                        "log_identical": hashlib.sha256(data).hexdigest() == spec["sha256"]}
        row["b200_over_reference"] = row["b200"]["steps_per_s"] / row["reference"]["steps_per_s"]
        out.append(row)
    return out


def dropin_scale(sizes=(64, 512, 4096, 32768), ticks: int = 40, warm: bool = True) -> list:
    """The drop-in crossover: the reference's own
    run_simulation over n sessions that all arrive at once (one long decode
    round each, no tools, a pool that holds them all, an admission window of
    n), so every tick plans over ~n ready sessions; `ticks` ticks
    (run_simulation's max_ticks guard ends the run) with MarsPolicy, then
    with the INTEGRATION.md binding.  ms per tick = wall / ticks."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref_dir) and ref_dir not in sys.path:
        sys.path.insert(1, ref_dir)
    try:
        from agentsched import baselines, control, sim, workload
    except ImportError:
        return [{"error": "agentsched (baseline/_ref) not importable"}]
    from paper_2604_26963_b200.admission import balance_and_admit as gpu_bna
    from paper_2604_26963_b200.policy import GpuMarsPolicy

    out = []
    # an untimed 64-session pass of both arms first: the process's first-use
    # costs (module loads, the first graph instantiations) are not per tick
    for n in ((64,) if warm else ()) + tuple(sizes):
        cfg = workload.RegimeConfig(mean_prompt_volume=2_000.0,
                                    prompt_volume_range=(1_000.0, 4_000.0), rounds_range=(1, 1),
                                    arrival_rate=1e6, request_count=n, seed=11,
                                    tool_duration_distribution=None,
                                    decode_tokens_range=(20_000, 30_000))
        traces = workload.generate_workload(cfg)
        params = sim.EngineParams(total_blocks=2_300 * n, tool_worker_slots=max(8, n))
        row = {"sessions": n, "ticks": ticks}
        for arm in ("reference", "b200"):
            pol = baselines.make_policy("mars") if arm == "reference" else \
                GpuMarsPolicy(max_sessions=max(n, 64))
            if arm == "b200":
                pol._engine()  # the device context: one-time setup, outside the timing
            orig = sim.balance_and_admit
            if arm == "b200":
                sim.balance_and_admit = gpu_bna
            t0 = time.perf_counter()
            try:
                sim.run_simulation(traces, params, pol,
                                   controller=control.ControllerConfig(initial_window=float(n)),
                                   max_ticks=ticks)
            except sim.SimulationStall:
                pass
            dt = time.perf_counter() - t0
            sim.balance_and_admit = orig
            if arm == "b200":
                pol.close()
            row[arm + "_ms_per_tick"] = dt * 1e3 / (ticks + 1)
        row["b200_over_reference"] = row["reference_ms_per_tick"] / row["b200_ms_per_tick"]
        if warm:
            warm = False  # (the untimed warm-up pass)
            continue
        out.append(row)
    return out


def cpu_reference(sessions: int, seed: int, reps: int = 1):
    """The reference's own step (agentsched from baseline/_ref, else the
    oracle port) over snapshot_v1(sessions) on one core; materialisation
    excluded."""
    from oracle.ref_step import timed_step
    from paper_2604_26963_b200.snapshot import snapshot_v1

    return [timed_step(snapshot_v1(sessions, seed=seed + r, pool="headroom")) for r in range(reps)]


_REF_SHARDS = []


def _ref_worker(j):
    from oracle.ref_step import timed_step
    return timed_step(_REF_SHARDS[j])


def workload_config(sessions: int, world: int) -> dict:
    """The `config` of both arms' lines (identical keys and values)."""
    return {"workload": "one MARS scheduling step over one global snapshot_v1 session table "
                        "(pin expiry, probe, control-plane admission, MLFQ aging, window "
                        "top-128, build_plan walk with reclamation, S2 retention, S5: the "
                        "pool ops of the step -- expired pins freed, the plan's allocs and "
                        "evictions; the B200 arm keeps every block's ID)"
                        + ("" if world == 1 else
                           f"; rows sharded rank mod {world} over data-parallel replicas"),
            "sessions": sessions, "pool": "headroom", "mix": "A",
            "parallelism": "1 replica" if world == 1 else
            f"{world} replicas: NCCL all-reduce of probe counters + all-gather of "
            "every admission entry (8 B each)",
            "l2": "flushed before every timed step (512 MiB scratch write); state restored "
                  "from a device checkpoint (untimed)"}


def run_reference_arm(a):
    """The reference's CPU path on every host core it can use, on the GPU
    arm's workload: snapshot_v1(sessions) split into P row-shards (row r ->
    shard r mod P), one process per shard running the real agentsched step
    (baseline/_ref; the oracle port if it is missing) over its shard
    concurrently; a step takes as long as the slowest shard (materialisation
    excluded), throughput = sessions / that time."""
    import multiprocessing as mp

    from oracle.ref_step import kind
    from paper_2604_26963_b200.snapshot import snapshot_shard, snapshot_v1

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", str(a.gpus)))
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    procs = max(1, min(a.ref_procs, cores)) if a.ref_procs > 0 else max(1, min(16, cores))
    snap = snapshot_v1(a.sessions, seed=0, pool="headroom")
    _REF_SHARDS[:] = [snapshot_shard(snap, procs, j) for j in range(procs)]
    times = []
    with mp.get_context("fork").Pool(procs) as pool:
        for i in range(a.warmup + a.steps):
            ts = pool.map(_ref_worker, range(procs))
            if i >= a.warmup:
                times.append(max(ts))
    per = sum(times) / len(times)
    val = a.sessions / per
    k = kind()
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "sessions/s",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": per * 1e3,
        "steps_per_s": 1.0 / per, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64+i64", "data": "synthetic (snapshot_v1, mix A, seed 0)",
        "config": workload_config(a.sessions, world),
        "cpu_baseline": {"value": val, "unit": "sessions/s", "cores": procs, "kind": k,
                         "sample": f"snapshot_v1({a.sessions}) in {procs} row-shards of "
                                   f"~{a.sessions // procs} sessions, one process per shard "
                                   "running " + ("the unmodified reference agentsched "
                                                 "(baseline/_ref)" if k == "reference" else
                                                 "the oracle port of agentsched")
                                   + " step (expiry, probe, refresh_pressure, balance_and_admit"
                                   " + admit, decide_retention on boundary rows, sorted ready "
                                   "list, MarsPolicy.plan_tick with the evictor); "
                                   "materialisation excluded; step time = slowest shard",
                         "host_cores": cores},
        "e2e": {"value": val, "unit": "sessions/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def advance_run(eng, snap, stream, flush, ticks):
    """SURVEY §8(f) row 1 measured: ``ticks`` consecutive whole ticks on the
    device from the 1M snapshot (MARS_MODE_ADVANCE: the scheduling step plus
    step_gpu / charge_service / every ending round's retention, pin or free),
    the control plane due every control_interval_s as in the reference loop.
    The state stays in HBM from tick to tick (no restore); each tick is timed
    with CUDA events around its graph launch, L2 flushed before it, and its
    outputs fetched after it (untimed).  The sequence is run once untimed
    first so every launch shape's graph is captured."""
    import torch

    from paper_2604_26963_b200 import _native as N
    cfg = eng.cfg
    tick = float(cfg.tick_duration_s)

    def run(timed):
        eng.restore()
        now, next_ctl = snap.now, snap.now
        out, evs = [], []
        wall.clear()
        for _ in range(ticks):
            due = now >= next_ctl - 1e-9
            if due:
                next_ctl = now + float(cfg.control_interval_s)
            si = eng.step_in(now, due, snap.active_tools, snap.queued_tools, snap.worker_slots,
                             N.MODE_ADVANCE)
            eng.flush_l2(flush)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            s0.record(stream)
            eng.enqueue(si)
            s1.record(stream)
            r = eng.fetch()
            wall.append(time.perf_counter() - w0)
            if r.status:
                raise SystemExit(f"advance tick status {r.status}")
            evs.append((s0, s1))
            out.append((due, int(r.total_tokens), len(r.end_rows), len(r.admitted_rows)))
            now = now + tick
        return [a.elapsed_time(b) for a, b in evs], out

    wall = []
    run(False)
    ms, out = run(True)
    eng.restore()
    ctl = [m for m, o in zip(ms, out) if o[0]]
    plain = [m for m, o in zip(ms, out) if not o[0]]
    return {"ticks": ticks, "sessions": snap.n, "ms_per_tick": sum(ms) / len(ms),
            "ms_per_tick_control": (sum(ctl) / len(ctl)) if ctl else None,
            "ms_per_tick_no_control": (sum(plain) / len(plain)) if plain else None,
            "ticks_per_s": 1e3 * len(ms) / sum(ms),
            # host view of the same ticks through the public API (step_in ->
            # graph launch -> fetch of the plan, journal and decisions)
            "wall_ms_per_tick": 1e3 * sum(wall) / len(wall),
            "tokens": sum(o[1] for o in out), "rounds_ended": sum(o[2] for o in out),
            "admitted": sum(o[3] for o in out),
            "timing": "CUDA events around each tick's graph launch, L2 flushed before each "
                      "tick, state resident in HBM across ticks"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--sessions", type=int, default=1_000_000)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-procs", type=int, default=0,
                    help="reference-arm processes (0: every host core, at most 16)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--flush-mb", type=int, default=512)
    ap.add_argument("--no-kv", action="store_true", help="skip the KV evict/restore sweep")
    ap.add_argument("--no-s5", dest="s5", action="store_false",
                    help="step without the block-ID manager (S5) attached")
    ap.add_argument("--no-dropin", dest="dropin", action="store_false",
                    help="skip the full-loop drop-in runs (configs 1 and 5)")
    ap.add_argument("--no-regimes", dest="regimes", action="store_false",
                    help="skip the heavy-reclaim / tick-grid regime sweep")
    ap.add_argument("--clock-load", type=int, default=100,
                    help="untimed 20-step batches run under the clock sampler first (0 under ncu)")
    ap.add_argument("--advance-ticks", type=int, default=40,
                    help="consecutive device-resident ticks (MARS_MODE_ADVANCE) to time; 0 = off")
    ap.add_argument("--hbm-sweep", default="100000,4000000,16000000,64000000",
                    help="table sizes for the size sweep: SURVEY config (2) at 100K, then beyond L2 (comma list, '' to skip)")
    a = ap.parse_args()
    if a.impl == "reference":
        return run_reference_arm(a)

    import numpy as np
    import torch

    from paper_2604_26963_b200.engine import MarsEngine, make_config, step_columns
    from paper_2604_26963_b200.snapshot import snapshot_v1

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # (validation only: MARS_BENCH_DEVICE pins every rank to one GPU and
    # MARS_BENCH_BACKEND=gloo replaces NCCL, so the sharded path can be
    # exercised end to end on a one-GPU box; never used for a bench number)
    if os.environ.get("MARS_BENCH_DEVICE") is not None:
        local = int(os.environ["MARS_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("MARS_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ONE global snapshot; with N ranks every rank
    # owns the rows r with r mod N == rank (strong scaling, the value counts
    # the global table's sessions once)
    snap = snapshot_v1(a.sessions, seed=0, pool="headroom")
    if world > 1:
        from paper_2604_26963_b200.snapshot import snapshot_shard
        snap = snapshot_shard(snap, world, rank, box_global=True)
    qcap = max(len(snap.queue), 1)
    qlens = [len(snap.queue)]
    if dist is not None:
        # the exchange buffers (1 + queue capacity words) must have the
        # same size on every rank: size them by the longest shard list
        ql = torch.tensor([len(snap.queue)], dtype=torch.int64, device="cuda")
        allq = [torch.zeros_like(ql) for _ in range(world)]
        dist.all_gather(allq, ql)
        qlens = [int(x.item()) for x in allq]
        qcap = max(max(qlens), 1)
    eng = MarsEngine(max_rows=snap.n, max_queue=qcap, device=local,
                     config=make_config(initial_window=snap.initial_window))
    eng.load_snapshot(snap)
    s5_blocks = None
    if a.s5:
        # S5 in the step: every session holding KV gets its block table (IDs
        # from a fresh pool, rank order); each step then frees the expired
        # pins' tables and applies the plan's alloc / evict journal on the
        # device (k_kv_exp_scan/push, k_kv_apply_step), state restored with
        # the table between steps
        from paper_2604_26963_b200.kvstore import KvBlockManager
        per_row = int(-(-(int(snap.cols["context"].max()) + 4096) // 16))
        kvm = KvBlockManager(eng, snap.total_blocks, max_blocks_per_row=per_row)
        s5_blocks = kvm.load_snapshot_tables(snap)
    si = eng.step_in(snap.now, True, snap.active_tools, snap.queued_tools, snap.worker_slots)
    flush = a.flush_mb << 20
    if world == 1:
        # a dedicated (non-default) stream: the step is captured as one CUDA
        # graph and the timing events are recorded on the stream it runs on
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        eng.lib.mars_set_stream(eng.ctx, stream.cuda_stream)
        eng.set_graph(True)

        def enqueue_step():
            eng.enqueue(si)
    else:
        # sharded replicas: every rank owns a 1M-session shard, the control
        # plane runs on NCCL-reduced counters and the all-gathered union list
        from paper_2604_26963_b200.dist import COUNTERS, ShardedEngine, exchange

        gpos = snap.meta["gpos"]
        sh = ShardedEngine(eng, world=world, rank=rank)
        stream = sh.stream
        torch.cuda.set_stream(stream)
        q = snap.queue
        sh.set_queue(q, snap.cols["req_blocks"][q], (snap.cols["flags"][q] & 16) != 0, gpos)

        def enqueue_step():
            sh.phase(si, 1)
            exchange(sh.xc[:len(COUNTERS)], sh.xsend, sh.xrecv)
            sh.phase(si, 2)
    eng.checkpoint()
    sharded_graph = None
    if world > 1 and os.environ.get("MARS_BENCH_BACKEND", "nccl") == "nccl":
        # the whole sharded step (phase 1, NCCL all-reduce + all-gather,
        # phase 2) as one CUDA graph; eager launches if the capture fails
        try:
            sh.capture(si)
            eng.restore()
            enqueue_step = sh.replay  # noqa: F811
            sharded_graph = True
        except Exception as exc:  # (reported in the line)
            sharded_graph = "eager: " + repr(exc)[:120]
            torch.cuda.synchronize()
            eng.restore()

    # correctness guard: one fetched step must succeed with status 0
    enqueue_step()
    res = eng.fetch()
    if res.status != 0:
        raise SystemExit(f"device step status {res.status}")
    eng.restore()

    for _ in range(a.warmup):
        enqueue_step()
        eng.restore()
    barrier()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    launches = 0
    with Clocks(local) as clk:
        # the K timed steps take a few ms, shorter than the sampler's 100 ms
        # period: keep the GPU on the same restore / flush / step load first
        # (a fixed count, identical on every rank: the sharded step runs
        # collectives) so the clock samples are taken under it (untimed)
        for _ in range(a.clock_load):
            for _ in range(20):
                eng.restore()
                eng.flush_l2(flush)
                enqueue_step()
            torch.cuda.synchronize()
        barrier()
        for i in range(a.steps):
            eng.restore()
            eng.flush_l2(flush)
            starts[i].record(stream)
            enqueue_step()           # N=1: one CUDA-graph launch per step
            ends[i].record(stream)
            launches += eng.launches()
        barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    dev_ms = sum(step_ms)
    t = torch.tensor([dev_ms], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / a.steps

    # per-kernel device times: CUDA events recorded by the library on the
    # stream each kernel runs on (stream launches: event timing is not
    # available inside graphs), same restore + L2 flush before every step
    eng.set_graph(False)
    eng.set_profiling(True)
    ktimes = []
    for i in range(a.steps):
        eng.restore()
        eng.flush_l2(flush)
        enqueue_step()
        ktimes.append(eng.kernel_times())
    eng.set_profiling(False)
    eng.set_graph(world == 1)
    kernel_ms = {k: statistics.median([kt[k] for kt in ktimes]) for k in ktimes[0]
                 if all(kt[k] >= 0 for kt in ktimes)}  # launched kernels only
    scan_avg = sum(kt["k_scan"] for kt in ktimes) / len(ktimes)

    # e2e: through the C ABI with host buffers: upload the table from pinned
    # host memory (every column this configuration's step reads,
    # engine.step_columns), run the step, fetch the plan/journal/decisions
    # The inputs live in the library's pinned input arena (mars_input_arena,
    # laid out like the device table): the upload is three pitched copies,
    # one per element-size group, instead of one copy per column
    names = step_columns(mode=si.mode)
    arena = eng.input_arena()
    for k in names:
        arena[k][:snap.n] = snap.cols[k]
    h2d = sum(snap.cols[k].nbytes for k in names)
    e2e_t = []
    d2h = 0
    e2e_warm = 3  # first copies out of freshly pinned pages are slower on some hosts
    e2e_up = []
    for i in range(a.e2e_steps + e2e_warm):
        eng.restore()
        eng.flush_l2(flush)
        barrier()
        t0 = time.perf_counter()
        eng.upsert_arena(snap.n, names)
        tu = time.perf_counter()
        enqueue_step()
        r = eng.fetch(copy=False)  # views of the pinned output arena (zero-copy)
        t1 = time.perf_counter()
        if i >= e2e_warm:
            e2e_t.append(t1 - t0)
            e2e_up.append(tu - t0)
        d2h = (r.expired_rows.nbytes * 2 + r.admitted_rows.nbytes + r.window_rows.nbytes
               + r.decode_rows.nbytes + r.prefill_rows.nbytes * 2 + r.evict_rows.nbytes * 3
               + r.journal_row.nbytes * 3 + r.ret_rows.nbytes * 7 + 4096)
    e2e_s = statistics.median(e2e_t)
    te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())

    # e2e_resident: the table stays in HBM between steps (as a serving
    # scheduler keeps it); every step uploads from pinned host memory the
    # rows that changed since the previous one -- modelled as 1 % of the
    # sessions, every column the step reads -- then runs the step and fetches
    # the plan / journal / decisions, all through the public API
    rng = np.random.default_rng(5)
    dn = max(1, snap.n // 100)
    drows = torch.from_numpy(np.sort(rng.choice(snap.n, dn, replace=False)).astype(np.int64)
                             ).pin_memory().numpy()
    dcols = {k: torch.from_numpy(np.ascontiguousarray(snap.cols[k][drows])).pin_memory().numpy()
             for k in names}
    dh2d = sum(v.nbytes for v in dcols.values()) + drows.nbytes
    res_t = []
    for i in range(a.e2e_steps + e2e_warm):
        eng.restore()
        eng.flush_l2(flush)
        barrier()
        t0 = time.perf_counter()
        eng.upsert(dcols, rows=drows)
        enqueue_step()
        r = eng.fetch(copy=False)
        t1 = time.perf_counter()
        if i >= e2e_warm:
            res_t.append(t1 - t0)
    res_s = statistics.median(res_t)
    tr_ = torch.tensor([res_s], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(tr_, op=dist.ReduceOp.MAX)
    res_s = float(tr_.item())

    adv = advance_run(eng, snap, stream, flush, a.advance_ticks) if (
        world == 1 and a.advance_ticks > 0) else None

    peak, peak_kind = _peaks()
    sb = scan_bytes(snap)
    achieved = sb / (scan_avg * 1e-3) / 1e9
    total_sessions = a.sessions
    steps_per_s = 1e3 / ms_per_step
    value = total_sessions * steps_per_s
    line = {
        "metric": METRIC, "value": value, "unit": "sessions/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
        "steps_per_s": steps_per_s, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64+i64",
        "data": "synthetic (snapshot_v1 mix A, seed 0" + (
            f", rows sharded rank mod {world})" if world > 1 else ")"),
        "config": workload_config(a.sessions, world),
        "s5_block_ids": s5_blocks,
        "roofline": {"bound": "hbm", "kernel": "k_scan", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": _ncu_traffic()[0],
                     "traffic_source": _ncu_traffic()[1],
                     "algorithmic_bytes": sb, "kernel_ms": scan_avg, "peak_source": peak_kind,
                     "step_algorithmic_bytes": step_bytes(snap),
                     "step_frac": step_bytes(snap) / (ms_per_step * 1e-3) / 1e9 / peak},
        "e2e": {"value": total_sessions / e2e_s, "unit": "sessions/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e2e_s * 1e3,
                "upload_ms": statistics.median(e2e_up) * 1e3,
                "inputs": "every column the step reads, all rows, uploaded each step from the pinned input arena (mars_upsert_arena: 3 pitched copies)"},
        "e2e_resident": {"value": total_sessions / res_s, "unit": "sessions/s",
                         "h2d_bytes_per_step": int(dh2d), "d2h_bytes_per_step": int(d2h),
                         "ms_per_step": res_s * 1e3,
                         "inputs": "table resident in HBM; 1 % of the rows (every column the "
                                   "step reads) uploaded each step"},
        "gpu_launches": launches,
        "sharded_graph": sharded_graph,
        "advance": adv,
        "kernel_ms_median": kernel_ms,
        "clocks": clk.summary(),
        "step_ms_min": min(step_ms), "step_ms_max": max(step_ms),
    }
    if not a.no_kv:
        try:
            line["kv"] = kv_sweep(local)
        except Exception as exc:  # the scheduler number stands on its own
            line["kv"] = {"error": repr(exc)[:300]}
        if rank == 0 and world == 1:
            try:
                line["kv_tier"] = kv_tier_run()
            except Exception as exc:
                line["kv_tier"] = {"error": repr(exc)[:300]}
    if rank == 0 and world == 1 and a.regimes:
        try:
            line["regimes"] = regime_sweep(local, a.sessions)
        except Exception as exc:  # the headline line stands on its own
            line["regimes"] = {"error": repr(exc)[:300]}
    if rank == 0 and world == 1 and a.dropin:
        try:
            line["dropin"] = dropin_sweep()
        except Exception as exc:  # the headline line stands on its own
            line["dropin"] = [{"error": repr(exc)[:300]}]
        try:
            line["dropin_scale"] = dropin_scale()
        except Exception as exc:
            line["dropin_scale"] = [{"error": repr(exc)[:300]}]
    if rank == 0 and world == 1 and a.hbm_sweep:
        try:
            line["hbm_sweep"] = hbm_sweep(local, [int(x) for x in a.hbm_sweep.split(",") if x])
        except Exception as exc:  # the headline line stands on its own
            line["hbm_sweep"] = {"error": repr(exc)[:300]}
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        from oracle.ref_step import kind as ref_kind
        t_cpu = cpu_reference(a.sessions, seed=0)[0]
        line["cpu_baseline"] = {
            "value": a.sessions / t_cpu, "unit": "sessions/s", "cores": 1, "kind": ref_kind(),
            "sample": f"one full step over snapshot_v1({a.sessions}) (the same table) with "
                      + ("the unmodified reference agentsched (baseline/_ref)"
                         if ref_kind() == "reference" else "the oracle port of agentsched")
                      + " on one core, materialisation excluded",
            "seconds": t_cpu}
    if rank == 0:
        print(json.dumps(line), flush=True)
    eng.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
