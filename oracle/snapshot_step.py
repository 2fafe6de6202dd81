"""Oracle for one scheduling step over a SoA snapshot.

Materialises the snapshot into the oracle's per-session objects, then runs
the reference tick's scheduling half in the reference order (sim.py:324-342):

1. expired pins, evicted in sorted session-id order (sim.py:324-325,
   baselines.py:396-399);
2. telemetry probe (sim.py:327);
3. if the control cadence is due: refresh_pressure, telemetry snapshot,
   balance_and_admit, admit() of every admitted entry (sim.py:329-337);
4. S2: decide_retention for every BOUNDARY row against the probe's
   telemetry (scheduler.py:190-213) -- boundary rows are DECODE rows, which
   neither expiry nor admission touch, and the decision is taken before the
   plan mutates anything;
5. MarsPolicy.plan_tick over the ready rows (baselines.py:440-455) with the
   sim's evictor (sim.py:168-188).

and returns every decision plus the full post-step state in canonical form
(row indices, not session-id strings).  TEST INFRASTRUCTURE ONLY.
"""

from __future__ import annotations

from typing import Dict, List, Optional

import numpy as np

from . import admission as adm
from .core import (DECODE, DONE, PREFILL, TOOL, WAITING_RESUME, BlockCounter, Clock, Journal,
                   Round, Session, TickModel, ceil_div, execute_tick, resume_cost, submit_round)
from .policy import MarsOracle, Mlfq, Pin, Prio, Retention, make_oracle_policy, retention

PHASES = ("waiting_admission", "prefill", "decode", "tool", "waiting_resume", "done")
PHASE_CODE = {p: i for i, p in enumerate(PHASES)}
F_ACTIVE, F_QUEUED, F_PINNED, F_BOUNDARY, F_LONG = 1, 2, 4, 8, 16


def sid_of(rank: int) -> str:
    return f"s{rank:07d}"


class World:
    """Objects materialised from a snapshot; ``row_of`` maps sid -> row."""

    def __init__(self, snap, enable_coordinator=True, enable_coscheduler=True,
                 mlfq: Optional[Mlfq] = None, controller: Optional[adm.Controller] = None,
                 pressure: Optional[adm.Pressure] = None,
                 ret: Optional[Retention] = None, policy: str = "mars") -> None:
        c = snap.cols
        n = snap.n
        self.snap = snap
        self.kind = policy
        if policy == "mars":
            self.policy = MarsOracle(mlfq=mlfq, ret=ret, pressure=pressure,
                                     enable_coordinator=enable_coordinator,
                                     enable_coscheduler=enable_coscheduler)
        elif policy in ("static_ttl", "dynamic_ttl"):
            self.policy = make_oracle_policy(policy, pressure=pressure)
        else:  # fcfs / program_priority: no pins, no MLFQ state; `served` is
            # Call.served_tokens (baselines.py:170-171)
            self.policy = make_oracle_policy(policy)
        self.pressure = getattr(self.policy, "pressure", None) or pressure or adm.Pressure()
        self.pool = BlockCounter(snap.total_blocks)
        self.gpu = TickModel()
        self.tel = adm.Counters(snap.total_blocks)
        self.tel.ema_tool_duration = snap.ema_tool
        self.tel.ema_blocks_per_session = snap.ema_blocks
        self.tel.blocks_seed = snap.blocks_seed
        for k, v in getattr(snap, "telemetry", {}).items():
            setattr(self.tel, k, v)
        self.ctl = controller or adm.Controller(initial_window=snap.initial_window)
        self.sessions: List[Session] = []
        self.row_of: Dict[str, int] = {}
        self.active: Dict[str, Session] = {}
        self.boundary: List[int] = []
        ph = c["phase"].tolist()
        fl = c["flags"].tolist()
        rank = c["rank"].tolist()
        ctx = c["context"].tolist()
        kv = c["kv"].tolist()
        rem = c["rem_decode"].tolist()
        r0p = c["r0_prefill"].tolist()
        r0d = c["r0_decode"].tolist()
        rs = c["ready_since"].tolist()
        ws = c["wait_since"].tolist()
        arr = c["arrival"].tolist()
        lv = c["level"].tolist()
        pr = c["promos"].tolist()
        sv = c["served"].tolist()
        dl = c["deadline"].tolist()
        pb = c["pinned_blocks"].tolist()
        plv = c["plevel"].tolist()
        pre = c["preempt"].tolist()
        rl = c["rounds_left"].tolist() if "rounds_left" in c else [0] * n
        alloc = self.pool.allocated
        pinned = self.pool.pinned
        used = 0
        for i in range(n):
            sid = sid_of(rank[i])
            rounds = [Round(r0p[i] if r0p[i] > 0 else 1, r0d[i] if r0d[i] > 0 else 1)]
            rounds += [Round(1, 1)] * int(rl[i])  # rounds after the current one
            s = Session(sid, rounds, arr[i])
            s.phase = PHASES[ph[i]] if ph[i] < 6 else "done"
            s.context_tokens = ctx[i]
            s.kv_tokens = kv[i]
            s.remaining_decode = rem[i]
            s.ready_since = rs[i]
            s.preemptions = pre[i]
            self.sessions.append(s)
            self.row_of[sid] = i
            self.policy.calls[sid] = s
            f = fl[i]
            if f & F_ACTIVE:
                self.active[sid] = s
                if policy == "mars":
                    self.policy.states[sid] = Prio(lv[i], lv[i], sv[i], ws[i], pr[i])
                else:
                    s.served_tokens = sv[i]
            if f & F_PINNED:
                s.pinned = True
                s.retention_deadline = dl[i]
                pinned[sid] = pb[i]
                used += pb[i]
                if hasattr(self.policy, "pinned"):
                    self.policy.pinned[sid] = Pin(sid, pb[i], 0.0, 0.0, dl[i], plv[i])
            elif kv[i] > 0:
                h = ceil_div(kv[i], 16)
                alloc[sid] = h
                used += h
            if f & F_BOUNDARY:
                self.boundary.append(i)
        self.pool.free_blocks = snap.total_blocks - used
        if self.pool.free_blocks != snap.free_blocks:
            raise ValueError("snapshot free_blocks inconsistent with its rows")
        self.queue: List[adm.Pending] = []
        for r in snap.queue.tolist():
            s = self.sessions[r]
            self.queue.append(adm.Pending(s, int(c["req_blocks"][r]),
                                          bool(fl[r] & F_LONG), 0.0))


class ToolCounts:
    def __init__(self, active: int, queued: int) -> None:
        self._a, self._q = active, queued

    def active_count(self) -> int:
        return self._a

    def queued_count(self) -> int:
        return self._q


def run_step(snap, control_due: bool = True, world: Optional[World] = None, **kw) -> dict:
    """One step; returns the canonical output dict (see module docstring)."""
    w = world or World(snap, **kw)
    pol, pool, tel, now = w.policy, w.pool, w.tel, snap.now
    log = Journal()
    row = w.row_of

    def observe(op, sid, n, from_pinned):
        log.emit(now, op, sid, blocks=n, from_pinned=bool(from_pinned))

    pool.observer = observe
    ops: List[tuple] = []

    def evict(sid, kind):
        s = pol.calls[sid]
        if kind == "pinned":
            n = pool.release_pinned(sid)
            s.pinned = False
            s.retention_deadline = None
        else:
            n = pool.free(sid)
        s.kv_tokens = 0
        if kind == "running":
            s.preemptions += 1
            if s.phase == DECODE:
                s.phase = PREFILL
        pol.on_evicted(sid)
        return n

    # 1. pin expiry
    expired = []
    for sid in pol.expired_pins(now):
        expired.append((row[sid], evict(sid, "pinned")))
    # 2. probe
    tel.probe(pool, ToolCounts(snap.active_tools, snap.queued_tools), len(w.active))
    probe = dict(available_kv=tel.available_kv, usage=tel.kv_usage_ratio,
                 active_sessions=tel.active_sessions)
    # 3. control plane
    control = None
    if control_due:
        adm.refresh_pressure(tel, w.pressure, snap.worker_slots)
        stats: dict = {}
        admitted = adm.admit_step(w.queue, w.ctl, tel, snap.worker_slots, w.pressure, now, None,
                                  stats)
        for e in admitted:
            s = e.call
            s.admit_time = now
            submit_round(s, now)
            tel.record("gpu_submit", {"projected_blocks": s.incremental_blocks(
                s.remaining_prefill, pool.block_size)})
            w.active[s.session_id] = s
            pol.on_admit(s, now)
        control = dict(w_adm=w.ctl.w_adm, last_update=w.ctl.last_update,
                       limit=stats["limit"], slots=stats["slots"],
                       admitted=[row[e.call.session_id] for e in admitted],
                       queue=[row[e.call.session_id] for e in w.queue],
                       cpu_overloaded=tel.cpu_overloaded, kv_overloaded=tel.kv_overloaded,
                       streaks=(tel.cpu_high_streak, tel.cpu_low_streak,
                                tel.kv_high_streak, tel.kv_low_streak),
                       blocks_seed=tel.blocks_seed, available_kv=tel.available_kv)
    # 4. S2 retention on boundary rows
    ret = []
    for r in w.boundary:
        if w.kind == "mars":
            d = retention(w.sessions[r], tel, pool, w.gpu, pol.retention, w.pressure, now)
        else:  # the policy's own rule; None = never pin (baselines.py:82-86)
            d = pol.retention_decision(w.sessions[r], pool, tel, w.gpu, now)
            if d is None:
                continue
        ret.append((r, d.pin, d.benefit_s, d.cost_s, d.retention_deadline))
    # 5. plan
    ready = [s for s in w.active.values() if s.phase in (PREFILL, DECODE)]
    ready.sort(key=lambda s: s.session_id)
    journal_start = len(log.records)

    def plan_evict(v):
        ops.append(("evict", row[v.session_id], v.kind))
        evict(v.session_id, v.kind)

    plan = pol.plan_tick(ready, pool, w.gpu, tel, now, plan_evict) if ready else None
    journal = [(r["kind"], row[r["session_id"]], r["blocks"], r["from_pinned"])
               for r in log.records[journal_start:]]
    exp_journal = [(r["kind"], row[r["session_id"]], r["blocks"], r["from_pinned"])
                   for r in log.records[:journal_start]]
    out = dict(
        expired=expired, expiry_journal=exp_journal, probe=probe, control=control,
        retention=ret,
        window=[row[s.session_id] for s in pol.last_window],
        decodes=[row[x] for x in plan.decode_ids] if plan else [],
        prefills=[(row[x], g) for x, g in plan.prefill_grants] if plan else [],
        evictions=[(row[v.session_id], v.kind, v.blocks) for v in plan.evictions] if plan else [],
        total_tokens=plan.total_tokens if plan else 0,
        journal=journal, free_blocks=pool.free_blocks, n_ready=len(ready),
    )
    out["state"] = extract_state(w)
    return out


def extract_state(w: World) -> Dict[str, np.ndarray]:
    """Post-step columns in snapshot layout."""
    n = len(w.sessions)
    st = {k: np.zeros(n, dtype=t) for k, t in (
        ("phase", np.uint8), ("flags", np.uint8), ("level", np.uint8), ("promos", np.uint8),
        ("wait_since", np.float64), ("ready_since", np.float64), ("context", np.int32),
        ("kv", np.int32), ("rem_decode", np.int32), ("preempt", np.int32),
        ("served", np.int64))}
    base_flags = w.snap.cols["flags"]
    ws0 = w.snap.cols["wait_since"]
    lv0 = w.snap.cols["level"]
    pr0 = w.snap.cols["promos"]
    sv0 = w.snap.cols["served"]
    queued = {w.row_of[e.call.session_id] for e in w.queue}
    for i, s in enumerate(w.sessions):
        st["phase"][i] = PHASE_CODE.get(s.phase, 5)
        f = int(base_flags[i]) & (F_BOUNDARY | F_LONG)
        if s.session_id in w.active:
            f |= F_ACTIVE
        if i in queued:
            f |= F_QUEUED
        if s.session_id in w.pool.pinned:
            f |= F_PINNED
        st["flags"][i] = f
        p = getattr(w.policy, "states", {}).get(s.session_id)
        if p is not None:
            st["level"][i], st["promos"][i] = p.level, p.promotions
            st["wait_since"][i], st["served"][i] = p.wait_since, p.served_tokens_at_level
        else:
            st["level"][i], st["promos"][i] = lv0[i], pr0[i]
            st["wait_since"][i], st["served"][i] = ws0[i], sv0[i]
        st["ready_since"][i] = s.ready_since
        st["context"][i] = s.context_tokens
        st["kv"][i] = s.kv_tokens
        st["rem_decode"][i] = s.remaining_decode
        st["preempt"][i] = s.preemptions
    return st


def finish_round(w: World, s: Session, now: float) -> None:
    """sim.py:233-279 without the event log and the tool plane (tools are the
    host's): note_round_blocks, DONE + free on the last round, else the
    policy's retention decision -- pin or free -- and phase TOOL."""
    sid = s.session_id
    pool, tel, pol = w.pool, w.tel, w.policy
    held = s.held_blocks(pool.block_size)
    tel.note_round_blocks(ceil_div(s.context_tokens, pool.block_size),
                          smoothing=w.pressure.ema_smoothing)
    if s.is_last_round:
        s.set_phase(DONE)
        pool.free(sid)
        s.kv_tokens = 0
        del w.active[sid]
        return
    d = pol.retention_decision(s, pool, tel, w.gpu, now)
    if d is not None and d.pin and held > 0:
        pool.pin(sid)
        s.pinned = True
        s.retention_deadline = d.retention_deadline
        pol.note_pin(s, d, held, now)
    else:
        pool.free(sid)
        s.kv_tokens = 0
    s.set_phase(TOOL)


def tool_return(w: World, s: Session, finish: float, duration: float, now: float) -> str:
    """The tool_end record's EMA fold (telemetry.py:96-120) and
    resume_from_tool (sim.py:190-231) on the World; returns warm / cold."""
    w.tel.record("tool_end", {"duration_s": duration}, smoothing=w.pressure.ema_smoothing)
    s.round_index += 1
    s.set_phase(WAITING_RESUME)
    warm = s.pinned and s.retention_deadline is not None and s.retention_deadline >= finish
    need = resume_cost(s, warm)
    if warm:
        w.pool.unpin(s.session_id)
        s.pinned = False
        s.retention_deadline = None
        w.policy.on_evicted(s.session_id)
    elif s.pinned:  # the pin expired between grid points: evicted at return
        w.pool.release_pinned(s.session_id)
        s.pinned = False
        s.retention_deadline = None
        s.kv_tokens = 0
        w.policy.on_evicted(s.session_id)
    submit_round(s, now)
    if s.remaining_prefill != need:
        raise ValueError("resume cost mismatch")
    w.policy.on_resume(s, now)
    return "warm" if warm else "cold"


def run_ticks(snap, ticks: int, control_ticks=(0,), resumes=None, **kw):
    """Consecutive ticks over one snapshot: each tick's scheduling half
    (run_step), then step_gpu on the plan (engine.py:459-514) and the tick's
    tail in progress order (sim.py:355-375: on_service, finish_round).  The
    clock advances by one tick per tick.  Returns each tick's canonical output
    (the last one carries the end-of-run table state) and the World."""
    w = World(snap, **kw)
    clock = Clock()
    clock.now = snap.now
    outs = []
    for k in range(ticks):
        snap.now = clock.now
        # tools that finished before this tick: (row, finish, duration,
        # next round's new prefill, its decode tokens), in finish order
        for (r, fin, dur, newp, dec) in (resumes or {}).get(k, []):
            s = w.sessions[r]
            s.rounds[s.round_index + 1] = Round(newp, dec)
            tool_return(w, s, fin, dur, clock.now)
        out = run_step(snap, control_due=k in control_ticks, world=w)
        out.pop("state")
        sess = w.sessions
        batch = [(sess[r], 0, True) for r in out["decodes"]]
        batch += [(sess[r], g, False) for r, g in out["prefills"]]
        prog = execute_tick(clock, w.gpu, batch)
        end = clock.now
        for (sid, pf, dd, _pdone, rdone) in prog:
            w.policy.on_service(sid, pf + dd, end)
            if rdone:
                finish_round(w, w.policy.calls[sid], end)
        outs.append(out)
    outs[-1]["state"] = extract_state(w)
    return outs, w
