"""Freeze golden fixtures from the REFERENCE implementation (dev container only).

Run:  python oracle/make_golden.py  [--ref /root/reference/pkg/src]

It imports the reference package ``agentsched`` (never shipped, never used at
run time) and writes under ``tests/golden/``:

* ``traces/<name>.jsonl``      -- the reference's generated parity traces
  (demo 64, 12-session fixture, criterion-7 80-session, 200-session faceoff,
  criterion-5 starvation run), frozen so no test regenerates them.
* ``sim_logs.json``            -- for every (trace, policy variant): record
  count + SHA-256 of the reference ``run_simulation`` event log serialised the
  way ``EventLog.dump_jsonl`` does (engine.py:95-98), plus the counters.
* ``sim_logs_baselines.json``  -- the same for the reference's comparison
  policies (fcfs, program_priority, static_ttl, dynamic_ttl) on four traces.
* ``snapshot_steps.json``      -- canonical outputs of one scheduling step
  computed with the reference's own objects/functions on small
  ``snapshot_v1`` instances (headroom, pressure, coordinator-off,
  coscheduler-off), in the same canonical form ``oracle/snapshot_step.py``
  emits.
* ``kat.json``                 -- known-answer vectors for the per-function
  mechanisms (retention, try_fit, reclaim, pack, AIMD, levels, charges).

TEST INFRASTRUCTURE ONLY.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import random
import sys
from dataclasses import replace

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
GOLDEN = os.path.join(REPO, "tests", "golden")


def _sha(events) -> str:
    h = hashlib.sha256()
    for r in events:
        h.update((json.dumps(r, separators=(",", ":")) + "\n").encode())
    return h.hexdigest()


def sim_cases(A):
    """(name, traces, EngineParams kwargs, run kwargs) -- reference test setups."""
    sys.path.insert(0, os.path.join(A.ref_root, "tests"))
    from helpers import R, tiny_regime, trace_of  # reference test helpers

    cases = []
    cases.append(("small12", A.generate_workload(tiny_regime()),
                  dict(total_blocks=4608, tool_worker_slots=4), {}))
    cases.append(("demo64", A.generate_workload(tiny_regime(64, seed=7)),
                  dict(total_blocks=4608, tool_worker_slots=4), {}))
    crit7 = A.RegimeConfig(
        mean_prompt_volume=9_000.0, prompt_volume_range=(1_000.0, 40_000.0),
        rounds_range=(1, 4), arrival_rate=1.5, request_count=80, seed=77,
        tool_duration_distribution={"family": "lognormal", "median_s": 4.0, "sigma": 0.9},
        decode_tokens_range=(32, 256), round0_volume_fraction=0.5)
    cases.append(("crit7_80", A.generate_workload(crit7),
                  dict(total_blocks=9_000, tool_worker_slots=8), {}))
    heavies = [trace_of(f"h{i:03d}", round(0.2 * i, 3), [R(2_000, 1)]) for i in range(300)]
    light = trace_of("light", 0.75, [R(4_096, 1)])
    starv = sorted(heavies + [light], key=lambda t: (t.arrival_time_s, t.session_id))
    cases.append(("starvation", starv, dict(total_blocks=100_000, tool_worker_slots=4),
                  {"enable_control_plane": False}))
    # faceoff (test_acceptance.py:70-131)
    tools = {"family": "constant", "value_s": 3.0}
    pops = (
        ("s", A.RegimeConfig(mean_prompt_volume=3_000.0, prompt_volume_range=(1_000.0, 8_000.0),
                             rounds_range=(2, 4), arrival_rate=20.0, request_count=110, seed=11,
                             tool_duration_distribution=tools, decode_tokens_range=(16, 64),
                             round0_volume_fraction=0.2), 0.0),
        ("w", A.RegimeConfig(mean_prompt_volume=20_000.0, prompt_volume_range=(8_000.0, 64_000.0),
                             rounds_range=(1, 2), arrival_rate=20.0, request_count=60, seed=64,
                             tool_duration_distribution=tools, decode_tokens_range=(16, 64),
                             round0_volume_fraction=0.6), 0.0),
        ("t", A.RegimeConfig(mean_prompt_volume=2_500.0, prompt_volume_range=(1_000.0, 8_000.0),
                             rounds_range=(2, 4), arrival_rate=0.06, request_count=30, seed=112,
                             tool_duration_distribution=tools, decode_tokens_range=(16, 64),
                             round0_volume_fraction=0.2), 12.0),
    )
    face = []
    for prefix, regime, off in pops:
        for t in A.generate_workload(regime):
            face.append(replace(t, session_id=prefix + t.session_id[1:],
                                arrival_time_s=t.arrival_time_s + off))
    face.sort(key=lambda t: (t.arrival_time_s, t.session_id))
    demand = sum(A.blocks_for_tokens(t.total_context_tokens, 16) for t in face)
    cases.append(("faceoff200", face, dict(total_blocks=int(0.30 * demand), tool_worker_slots=64),
                  {"controller": dict(initial_window=96.0)}))
    # OpenHands-style heavy preset with CPU tool-slot pressure (BASELINE configs[4])
    heavy = A.regime_preset("heavy", arrival_rate=0.5, request_count=40, seed=5)
    htr = A.generate_workload(heavy)
    hdemand = sum(A.blocks_for_tokens(t.total_context_tokens, 16) for t in htr)
    hbig = max(A.blocks_for_tokens(t.total_context_tokens, 16) for t in htr)
    cases.append(("openhands_heavy40", htr,
                  dict(total_blocks=max(int(0.30 * hdemand), hbig), tool_worker_slots=8), {}))
    return cases


VARIANTS = {
    "mars": dict(),
    "mars-no-coordinator": dict(enable_coordinator=False),
    "mars-no-coscheduler": dict(enable_coscheduler=False),
}


def freeze_sims(A, out):
    os.makedirs(os.path.join(GOLDEN, "traces"), exist_ok=True)
    logs = {}
    for name, traces, pkw, rkw in sim_cases(A):
        path = os.path.join(GOLDEN, "traces", f"{name}.jsonl")
        A.save_trace(traces, path)
        variants = ["mars"] if name in ("starvation",) else list(VARIANTS) + ["mars-no-control"]
        if name == "openhands_heavy40":
            variants = ["mars"]
        for v in variants:
            pol = A.make_policy("mars", **VARIANTS.get(v, {}))
            kw = dict(rkw)
            if v == "mars-no-control":
                kw["enable_control_plane"] = False
            if "controller" in kw:
                kw["controller"] = A.ControllerConfig(**kw["controller"])
            res = A.run_simulation(A.load_trace(path), A.EngineParams(**pkw), pol, **kw)
            key = f"{name}/{v}"
            logs[key] = dict(trace=f"traces/{name}.jsonl", engine=pkw,
                             run={k: (v2 if k != "controller" else rkw["controller"])
                                  for k, v2 in kw.items()},
                             variant=VARIANTS.get(v, {}), records=len(res.events),
                             sha256=_sha(res.events), counters=res.counters,
                             horizon_s=res.horizon_s)
            print(f"  {key}: {len(res.events)} records")
    out["sim_logs.json"] = logs


BASELINE_KINDS = ("fcfs", "program_priority", "static_ttl", "dynamic_ttl")
BASELINE_TRACES = ("small12", "demo64", "crit7_80", "faceoff200")


def freeze_baseline_sims(A, out):
    """The reference's four comparison policies (baselines.py:108-315) on the
    frozen traces: record count, SHA-256 and counters of each event log."""
    logs = {}
    for name, traces, pkw, rkw in sim_cases(A):
        if name not in BASELINE_TRACES:
            continue
        path = os.path.join(GOLDEN, "traces", f"{name}.jsonl")
        for kind in BASELINE_KINDS:
            kw = dict(rkw)
            if "controller" in kw:
                kw["controller"] = A.ControllerConfig(**kw["controller"])
            res = A.run_simulation(A.load_trace(path), A.EngineParams(**pkw),
                                   A.make_policy(kind), **kw)
            key = f"{name}/{kind}"
            logs[key] = dict(trace=f"traces/{name}.jsonl", engine=pkw,
                             run={k: (v2 if k != "controller" else rkw["controller"])
                                  for k, v2 in kw.items()},
                             policy=kind, records=len(res.events), sha256=_sha(res.events),
                             counters=res.counters, horizon_s=res.horizon_s)
            print(f"  {key}: {len(res.events)} records")
    out["sim_logs_baselines.json"] = logs


# ---------------------------------------------------------------------------
# Snapshot step through the reference's own objects
# ---------------------------------------------------------------------------

PHASES = ("waiting_admission", "prefill", "decode", "tool", "waiting_resume", "done")
F_ACTIVE, F_QUEUED, F_PINNED, F_BOUNDARY, F_LONG = 1, 2, 4, 8, 16


def ref_snapshot_step(A, snap, enable_coordinator=True, enable_coscheduler=True, policy="mars",
                      control_due=True):
    """One scheduling step through the reference's own objects (any of its
    policies, baselines.py:108-455), canonical output as oracle/snapshot_step.py."""
    import numpy as np
    from agentsched.scheduler import PinnedSession, PriorityState, RetentionConfig, decide_retention
    from agentsched.telemetry import refresh_pressure

    c = snap.cols
    n = snap.n
    mars = policy == "mars"
    pol = A.make_policy(policy, enable_coordinator=enable_coordinator,
                        enable_coscheduler=enable_coscheduler)
    pool = A.KvPool(total_blocks=snap.total_blocks)
    gpu = A.GpuModel()
    tel = A.Telemetry(total_blocks=snap.total_blocks)
    tel.ema_tool_duration = snap.ema_tool
    tel.ema_blocks_per_session = snap.ema_blocks
    tel.blocks_seed = snap.blocks_seed
    ctl = A.ControllerState(config=A.ControllerConfig(initial_window=snap.initial_window))
    pressure = A.PressureConfig()
    sess, row, active, boundary = [], {}, {}, []
    used = 0
    for i in range(n):
        sid = f"s{int(c['rank'][i]):07d}"
        r0p, r0d = int(c["r0_prefill"][i]), int(c["r0_decode"][i])
        call = A.Call(session_id=sid, rounds=[A.RoundSpec(max(r0p, 1), max(r0d, 1))],
                      arrival_time=float(c["arrival"][i]))
        call.phase = A.Phase(PHASES[int(c["phase"][i])])
        call.context_tokens = int(c["context"][i])
        call.kv_tokens = int(c["kv"][i])
        call.remaining_decode = int(c["rem_decode"][i])
        call.ready_since = float(c["ready_since"][i])
        call.preemptions = int(c["preempt"][i])
        sess.append(call)
        row[sid] = i
        pol.register_call(call)
        f = int(c["flags"][i])
        if f & F_ACTIVE:
            active[sid] = call
            lv = int(c["level"][i])
            if mars:
                pol.states[sid] = PriorityState(level=lv, base_level=lv,
                                                served_tokens_at_level=int(c["served"][i]),
                                                wait_since=float(c["wait_since"][i]),
                                                promotions=int(c["promos"][i]))
            else:  # Call.served_tokens (program_priority's key, baselines.py:170-171)
                call.served_tokens = int(c["served"][i])
        if f & F_PINNED:
            call.pinned = True
            call.retention_deadline = float(c["deadline"][i])
            pb = int(c["pinned_blocks"][i])
            pool.pinned[sid] = pb
            used += pb
            pol.pinned[sid] = PinnedSession(sid, pb, 0.0, 0.0, float(c["deadline"][i]),
                                            int(c["plevel"][i]) if mars else 0)
        elif call.kv_tokens > 0:
            h = A.blocks_for_tokens(call.kv_tokens, 16)
            pool.allocated[sid] = h
            used += h
        if f & F_BOUNDARY:
            boundary.append(i)
    pool.free_blocks = snap.total_blocks - used
    assert pool.free_blocks == snap.free_blocks
    queue = [A.QueueEntry(call=sess[r], req_blocks=int(c["req_blocks"][r]),
                          is_long_session=bool(int(c["flags"][r]) & F_LONG), enqueue_time=0.0)
             for r in snap.queue.tolist()]
    records = []
    pool.observer = lambda op, sid, b, fp: records.append((op, row[sid], b, bool(fp)))
    now = snap.now

    def evict(sid, kind):
        call = pol.calls[sid]
        if kind == "pinned":
            b = pool.release_pinned(sid)
            call.pinned = False
            call.retention_deadline = None
        else:
            b = pool.free(sid)
        call.kv_tokens = 0
        if kind == "running":
            call.preemptions += 1
            if call.phase == A.Phase.DECODE:
                call.set_phase(A.Phase.PREFILL)
        pol.on_evicted(sid)
        return b

    expired = [(row[s], evict(s, "pinned")) for s in pol.expired_pins(now)]
    exp_journal = list(records)

    class Plane:
        worker_slots = snap.worker_slots

        def active_count(self):
            return snap.active_tools

        def queued_count(self):
            return snap.queued_tools

    tel.probe(pool, Plane(), active_sessions=len(active))
    probe = dict(available_kv=tel.available_kv, usage=tel.kv_usage_ratio,
                 active_sessions=tel.active_sessions)
    control = None
    if control_due:
        refresh_pressure(tel, pressure, snap.worker_slots)
        clock = A.SimClock()
        clock.now = now
        log = A.EventLog()
        admitted = A.balance_and_admit(queue, ctl, tel, snap.worker_slots, pressure, clock, log)
        wu = log.records[-1]
        for e in admitted:
            call = e.call
            call.admit_time = now
            A.submit_round(call, now)
            tel.record("gpu_submit", {"projected_blocks": call.incremental_blocks(
                call.remaining_prefill, pool.block_size)})
            active[call.session_id] = call
            pol.on_admit(call, now)
        control = dict(w_adm=ctl.w_adm, last_update=ctl.last_update, limit=wu["limit"],
                       slots=wu["slots"], admitted=[row[e.call.session_id] for e in admitted],
                       queue=[row[e.call.session_id] for e in queue],
                       cpu_overloaded=tel.cpu_overloaded, kv_overloaded=tel.kv_overloaded,
                       streaks=[tel.cpu_high_streak, tel.cpu_low_streak, tel.kv_high_streak,
                                tel.kv_low_streak],
                       blocks_seed=tel.blocks_seed, available_kv=tel.available_kv)
    ret = []
    for r in boundary:
        if mars:
            d = decide_retention(sess[r], tel, pool, gpu, RetentionConfig(), pressure, now)
        else:  # the policy's own rule; None = never pin (baselines.py:82-86)
            d = pol.retention_decision(sess[r], pool, tel, gpu, now)
            if d is None:
                continue
        ret.append([r, d.pin, d.benefit_s, d.cost_s, d.retention_deadline])
    ready = sorted((x for x in active.values() if x.phase in (A.Phase.PREFILL, A.Phase.DECODE)),
                   key=lambda x: x.session_id)
    window_holder = []

    # capture the window exactly as build_plan forms it (scheduler.py:310, the
    # scheduler module's only sorted() call)
    def plan_tick_capture():
        import agentsched.scheduler as S
        real_sorted = sorted

        def spy(seq, key=None):
            out = real_sorted(seq, key=key)
            if not window_holder:
                window_holder.append(out[:128])
            return out
        S.sorted = spy
        try:
            return pol.plan_tick(ready, pool, gpu, tel, now,
                                 lambda v: evict(v.session_id, v.kind))
        finally:
            del S.sorted

    start = len(records)
    plan = plan_tick_capture() if ready else None
    journal = records[start:]
    win = window_holder[0] if window_holder else []
    st = {}
    cols = {k: [] for k in ("phase", "flags", "level", "promos", "wait_since", "ready_since",
                            "context", "kv", "rem_decode", "preempt", "served")}
    queued = {row[e.call.session_id] for e in queue}
    for i, call in enumerate(sess):
        cols["phase"].append(PHASES.index(call.phase.value))
        f = int(c["flags"][i]) & (F_BOUNDARY | F_LONG)
        if call.session_id in active:
            f |= F_ACTIVE
        if i in queued:
            f |= F_QUEUED
        if call.session_id in pool.pinned:
            f |= F_PINNED
        cols["flags"].append(f)
        p = pol.states.get(call.session_id) if mars else None
        if p is not None:
            cols["level"].append(p.level)
            cols["promos"].append(p.promotions)
            cols["wait_since"].append(p.wait_since)
            cols["served"].append(p.served_tokens_at_level)
        else:
            cols["level"].append(int(c["level"][i]))
            cols["promos"].append(int(c["promos"][i]))
            cols["wait_since"].append(float(c["wait_since"][i]))
            cols["served"].append(int(c["served"][i]))
        cols["ready_since"].append(call.ready_since)
        cols["context"].append(call.context_tokens)
        cols["kv"].append(call.kv_tokens)
        cols["rem_decode"].append(call.remaining_decode)
        cols["preempt"].append(call.preemptions)
    dtypes = dict(phase=np.uint8, flags=np.uint8, level=np.uint8, promos=np.uint8,
                  wait_since=np.float64, ready_since=np.float64, context=np.int32, kv=np.int32,
                  rem_decode=np.int32, preempt=np.int32, served=np.int64)
    for k, v in cols.items():
        st[k] = hashlib.sha256(np.asarray(v, dtype=dtypes[k]).tobytes()).hexdigest()
    return dict(
        expired=expired, expiry_journal=exp_journal, probe=probe, control=control,
        retention=ret, window=[row[x.session_id] for x in win],
        decodes=[row[x] for x in plan.decode_ids] if plan else [],
        prefills=[[row[x], g] for x, g in plan.prefill_grants] if plan else [],
        evictions=[[row[v.session_id], v.kind, v.blocks] for v in plan.evictions] if plan else [],
        total_tokens=plan.total_tokens if plan else 0, journal=journal,
        free_blocks=pool.free_blocks, n_ready=len(ready), state_sha256=st)


SNAP_CASES = [
    dict(n=2000, seed=1, pool="headroom"),
    dict(n=2000, seed=2, pool="pressure"),
    dict(n=3000, seed=3, pool="pressure", enable_coordinator=False),
    dict(n=3000, seed=4, pool="pressure", enable_coscheduler=False),
    dict(n=1500, seed=5, pool="headroom", enable_coordinator=False),
    dict(n=20000, seed=6, pool="headroom"),
    dict(n=20000, seed=7, pool="pressure"),
]


def freeze_snapshots(A, out):
    sys.path.insert(0, REPO)
    from paper_2604_26963_b200.snapshot import snapshot_v1

    res = []
    for case in SNAP_CASES:
        kw = {k: case[k] for k in ("enable_coordinator", "enable_coscheduler") if k in case}
        snap = snapshot_v1(case["n"], seed=case["seed"], pool=case["pool"])
        o = ref_snapshot_step(A, snap, **kw)
        res.append(dict(case=case, out=json.loads(json.dumps(o))))
        print(f"  snapshot {case}: window {len(o['window'])} evictions {len(o['evictions'])} "
              f"admitted {len(o['control']['admitted'])}")
    out["snapshot_steps.json"] = res


# heavy-reclaim and tick-gridded snapshots (tests/_variants.py): steps that
# take dozens of victims per claim sequence, all five policies, exact time ties
HEAVY_CASES = [
    dict(n=30_000, seed=81, kind="reclaim_heavy", policy=p, grid=g)
    for p in ("mars", "fcfs", "program_priority", "static_ttl", "dynamic_ttl")
    for g in (False, True)
] + [
    dict(n=30_000, seed=82, kind="tick_grid", policy="mars", grid=True),
    dict(n=30_000, seed=83, kind="reclaim_heavy", policy="mars", grid=True,
         enable_coordinator=False),
]


def heavy_snapshot(case):
    sys.path.insert(0, REPO)
    from paper_2604_26963_b200.snapshot import snapshot_v1
    from tests._variants import reclaim_heavy, tick_grid

    if case["kind"] == "reclaim_heavy":
        snap = reclaim_heavy(case["n"], case["seed"], case["policy"])
    else:
        snap = snapshot_v1(case["n"], seed=case["seed"], pool="pressure")
    if case.get("grid"):
        snap = tick_grid(snap, case["seed"])
    return snap


def heavy_kw(case):
    kw = {k: case[k] for k in ("enable_coordinator", "enable_coscheduler") if k in case}
    kw["policy"] = case["policy"]
    kw["control_due"] = case["policy"] == "mars"
    return kw


def freeze_heavy(A, out):
    res = []
    for case in HEAVY_CASES:
        snap = heavy_snapshot(case)
        o = ref_snapshot_step(A, snap, **heavy_kw(case))
        res.append(dict(case=case, out=json.loads(json.dumps(o))))
        print(f"  heavy {case}: evictions {len(o['evictions'])} "
              f"(pinned {sum(1 for e in o['evictions'] if e[1] == 'pinned')})")
    out["heavy_steps.json"] = res


# ---------------------------------------------------------------------------
# Known-answer vectors
# ---------------------------------------------------------------------------


def freeze_kat(A, out):
    from agentsched import control as C
    from agentsched import scheduler as S
    from agentsched.telemetry import PressureConfig, Telemetry, refresh_pressure

    rng = random.Random(2604)
    kat = {}
    # retention (scheduler.py:190-213) incl. the reference test's examples
    rows = []
    for _ in range(400):
        total = rng.randrange(1, 1_000_000)
        kv = rng.randrange(0, 262_144)
        ctx = kv + rng.randrange(0, 4096)
        u = rng.choice([0.0, 0.5, 0.7, 0.9, 0.99, 1.0, 1.2, rng.random()])
        ema = rng.choice([None, 0.0, 1.5, 5.0, 30.0, 59.9, 60.0, 61.0, rng.uniform(0, 100)])
        now = rng.choice([0.0, 12.25, 1000.0, rng.uniform(0, 5000)])
        call = A.Call(session_id="x", rounds=[A.RoundSpec(1, 1)], arrival_time=0.0)
        call.context_tokens, call.kv_tokens = ctx, kv
        tel = Telemetry(total_blocks=total)
        tel.kv_usage_ratio = u
        tel.ema_tool_duration = ema
        pool = A.KvPool(total_blocks=total)
        d = S.decide_retention(call, tel, pool, A.GpuModel(), S.RetentionConfig(),
                               PressureConfig(), now)
        rows.append(dict(total=total, kv=kv, ctx=ctx, usage=u, ema=ema, now=now, pin=d.pin,
                         benefit=d.benefit_s, cost=d.cost_s, deadline=d.retention_deadline))
    kat["retention"] = rows
    # try_fit (scheduler.py:136-157)
    rows = []
    for _ in range(2000):
        total = rng.randrange(1, 400)
        kv = rng.randrange(0, total * 16 + 1)
        held = A.blocks_for_tokens(kv, 16)
        if held > total:
            continue
        other = rng.randrange(0, total - held + 1)
        desired = rng.randrange(1, 3000)
        pool = A.KvPool(total_blocks=total)
        if held:
            pool.allocate("self", held)
        if other:
            pool.allocate("other", other)
        call = A.Call(session_id="self", rounds=[A.RoundSpec(1, 1)], arrival_time=0.0)
        call.kv_tokens = call.context_tokens = kv
        free = pool.free_blocks
        g = S.try_fit(call, desired, pool)
        rows.append(dict(kv=kv, desired=desired, free=free, grant=g))
    kat["try_fit"] = rows
    # pack_queue (control.py:101-122)
    rows = []
    for _ in range(300):
        n = rng.randrange(0, 30)
        reqs = [rng.randrange(1, 200) for _ in range(n)]
        longs = [rng.random() < 0.8 for _ in range(n)]
        if rng.random() < 0.3:
            longs = [True] * n
        cpu = rng.random() < 0.3
        avail = rng.randrange(0, 2000)
        tel = Telemetry(total_blocks=10_000)
        tel.cpu_overloaded = cpu
        tel.available_kv = avail
        q = [A.QueueEntry(call=A.Call(session_id=f"q{i:03d}", rounds=[A.RoundSpec(1, 1)],
                                      arrival_time=0.0), req_blocks=r, is_long_session=lg,
                          enqueue_time=0.0) for i, (r, lg) in enumerate(zip(reqs, longs))]
        order = C.pack_queue(q, tel)
        rows.append(dict(reqs=reqs, longs=longs, cpu=cpu, avail=avail,
                         order=[int(e.call.session_id[1:]) for e in order]))
    kat["pack"] = rows
    # balance_and_admit replay over a pressure trace (control.py:141-208, telemetry.py:174-208)
    rows = []
    tel = Telemetry(total_blocks=50_000)
    st = C.ControllerState(config=C.ControllerConfig())
    pc = PressureConfig()
    steps = []
    now = 0.0
    for i in range(500):
        now += rng.choice([0.5, 1.0, 2.0, 2.0, 3.0])
        tel.active_tools = rng.randrange(0, 12)
        tel.queued_tools = rng.choice([0, 0, 0, rng.randrange(0, 5)])
        tel.kv_usage_ratio = rng.random()
        tel.available_kv = rng.randrange(0, 50_000)
        tel.active_sessions = rng.randrange(0, 40)
        if rng.random() < 0.1:
            tel.note_round_blocks(rng.randrange(1, 3000))
        refresh_pressure(tel, pc, 8)
        q = [A.QueueEntry(call=A.Call(session_id=f"q{k:03d}", rounds=[A.RoundSpec(1, 1)],
                                      arrival_time=0.0), req_blocks=rng.randrange(1, 5000),
                          is_long_session=False, enqueue_time=0.0)
             for k in range(rng.randrange(0, 12))]
        reqs = [e.req_blocks for e in q]
        clock = A.SimClock()
        clock.now = now
        adm = C.balance_and_admit(q, st, tel, 8, pc, clock, None)
        steps.append(dict(now=now, active_tools=tel.active_tools, queued_tools=tel.queued_tools,
                          usage=tel.kv_usage_ratio, avail=tel.available_kv,
                          active=tel.active_sessions, ema_blocks=tel.ema_blocks_per_session,
                          reqs=reqs, cpu=tel.cpu_overloaded, kvo=tel.kv_overloaded,
                          w=st.w_adm, admitted=[int(e.call.session_id[1:]) for e in adm],
                          seed=tel.blocks_seed))
    kat["admit_replay"] = steps
    # reclaim_for (scheduler.py:228-267)
    rows = []
    for _ in range(300):
        total = 10_000
        pool = A.KvPool(total_blocks=total)
        pins, run = {}, []
        lv = {}
        for k in range(rng.randrange(0, 8)):
            sid = f"p{k}"
            b = rng.randrange(1, 50)
            pool.allocate(sid, b)
            pool.pin(sid)
            pins[sid] = S.PinnedSession(sid, b, 0.0, 0.0, rng.uniform(0, 20), rng.randrange(0, 4))
        for k in range(rng.randrange(0, 8)):
            sid = f"r{k}"
            kv = rng.randrange(0, 800)
            call = A.Call(session_id=sid, rounds=[A.RoundSpec(1, 1)], arrival_time=0.0)
            call.kv_tokens = kv
            if kv:
                pool.allocate(sid, A.blocks_for_tokens(kv, 16))
            run.append(call)
            lv[sid] = rng.randrange(0, 4)
        filler = pool.free_blocks - rng.randrange(0, 40)
        if filler > 0:
            pool.allocate("fill", filler)
        need = rng.randrange(1, 200)
        now = 10.0
        vs = S.reclaim_for(need, pool, pins, run, lambda c: lv[c.session_id], now)
        rows.append(dict(free=pool.free_blocks, need=need, now=now,
                         pins=[[p.session_id, p.pinned_blocks, p.retention_deadline, p.level]
                               for p in pins.values()],
                         running=[[c.session_id, c.kv_tokens, lv[c.session_id]] for c in run],
                         victims=[[v.session_id, v.kind, v.blocks] for v in vs]))
    kat["reclaim"] = rows
    # levels and charges (scheduler.py:87-108)
    kat["initial_level"] = [[t, S.initial_level(t, S.MlfqConfig())]
                            for t in [1, 3999, 4000, 4001, 31999, 32000, 32001, 127999, 128000,
                                      128001, 262144] + [rng.randrange(1, 262144) for _ in range(50)]]
    rows = []
    for _ in range(200):
        charges = [rng.randrange(0, 5000) for _ in range(rng.randrange(0, 30))]
        ps = S.PriorityState(level=rng.randrange(0, 4), base_level=0)
        start = ps.level
        for ch in charges:
            S.charge_service(ps, ch, S.MlfqConfig())
        rows.append(dict(start=start, charges=charges, level=ps.level,
                         served=ps.served_tokens_at_level))
    kat["charge"] = rows
    out["kat.json"] = kat


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--only", default="")
    a = ap.parse_args(argv)
    sys.path.insert(0, a.ref)
    import agentsched as A
    A.ref_root = os.path.dirname(a.ref)
    out = {}
    only = set(filter(None, a.only.split(",")))
    if not only or "sims" in only:
        freeze_sims(A, out)
    if not only or "baselines" in only:
        freeze_baseline_sims(A, out)
    if not only or "snapshots" in only:
        freeze_snapshots(A, out)
    if not only or "kat" in only:
        freeze_kat(A, out)
    if not only or "heavy" in only:
        freeze_heavy(A, out)
    os.makedirs(GOLDEN, exist_ok=True)
    for name, obj in out.items():
        with open(os.path.join(GOLDEN, name), "w") as fh:
            json.dump(obj, fh, separators=(",", ":"), sort_keys=False)
        print("wrote", name)


if __name__ == "__main__":
    main()
