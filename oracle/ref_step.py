"""The reference's own scheduling step over a snapshot, for the CPU timings.

``bench.py --impl reference`` (and the ``cpu_baseline`` leg of the default
line) time the REAL reference package ``agentsched`` -- installed, unmodified,
into ``baseline/_ref`` -- on the same synthetic session table the
device step runs over.  ``RefStep`` materialises a snapshot into the
reference's objects (``Call``, ``PriorityState``, ``PinnedSession``,
``KvPool``, ``Telemetry``, ``ControllerState``, ``QueueEntry``; untimed) and
``run()`` executes one tick's scheduling half exactly as ``sim.py:324-342``
orders it:

1. ``MarsPolicy.expired_pins`` + the evictor (sim.py:324-325, 168-188);
2. ``Telemetry.probe`` (sim.py:327);
3. ``refresh_pressure`` + ``balance_and_admit`` + ``admit`` (sim.py:329-337,
   148-166; control.py:166-208);
4. ``decide_retention`` for the boundary rows (scheduler.py:190-213);
5. ``MarsPolicy.plan_tick`` (baselines.py:440-455: promote_waiting +
   build_plan with the reclaimer) with the sim's evictor.

When ``baseline/_ref`` is not importable the oracle port (``oracle/``) stands
in (``kind() == "port"``).  TEST / BENCH INFRASTRUCTURE ONLY: never imported by
the product package.
"""

from __future__ import annotations

import os
import sys
from typing import Optional

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
REF_DIR = os.path.join(REPO, "baseline", "_ref")

PHASES = ("waiting_admission", "prefill", "decode", "tool", "waiting_resume", "done")
F_ACTIVE, F_QUEUED, F_PINNED, F_BOUNDARY, F_LONG = 1, 2, 4, 8, 16

_A = None


def agentsched():
    """The installed reference package, or None."""
    global _A
    if _A is None:
        if os.path.isdir(REF_DIR) and REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        try:
            import agentsched as A  # noqa: F401
            from agentsched import baselines  # noqa: F401
            _A = A
        except Exception:
            _A = False
    return _A or None


def kind() -> str:
    return "reference" if agentsched() is not None else "port"


class RefStep:
    """One snapshot materialised into the reference's objects (untimed)."""

    def __init__(self, snap, control_due: bool = True, policy: str = "mars") -> None:
        A = agentsched()
        if A is None:
            from oracle.snapshot_step import World
            self.port = World(snap, policy=policy)
            self.snap = snap
            self.control_due = control_due
            return
        self.port = None
        from agentsched.scheduler import PinnedSession, PriorityState

        self.A = A
        c = snap.cols
        n = snap.n
        self.snap = snap
        self.control_due = control_due
        self.mars = policy == "mars"
        pol = A.make_policy(policy)
        pool = A.KvPool(total_blocks=snap.total_blocks)
        tel = A.Telemetry(total_blocks=snap.total_blocks)
        tel.ema_tool_duration = snap.ema_tool
        tel.ema_blocks_per_session = snap.ema_blocks
        tel.blocks_seed = snap.blocks_seed
        for k, v in getattr(snap, "telemetry", {}).items():
            setattr(tel, k, v)
        self.ctl = A.ControllerState(config=A.ControllerConfig(initial_window=snap.initial_window))
        self.pressure = A.PressureConfig()
        self.gpu = A.GpuModel()
        sess, active, boundary = [], {}, []
        used = 0
        cols = {k: c[k].tolist() for k in ("rank", "r0_prefill", "r0_decode", "arrival", "phase",
                                           "context", "kv", "rem_decode", "ready_since",
                                           "preempt", "flags", "level", "served", "wait_since",
                                           "promos", "deadline", "pinned_blocks", "plevel",
                                           "req_blocks")}
        Phase = A.Phase
        phases = [Phase(p) for p in PHASES]
        for i in range(n):
            sid = f"s{cols['rank'][i]:07d}"
            call = A.Call(session_id=sid,
                          rounds=[A.RoundSpec(max(cols["r0_prefill"][i], 1),
                                              max(cols["r0_decode"][i], 1))],
                          arrival_time=cols["arrival"][i])
            call.phase = phases[cols["phase"][i]] if cols["phase"][i] < 6 else Phase.DONE
            call.context_tokens = cols["context"][i]
            call.kv_tokens = cols["kv"][i]
            call.remaining_decode = cols["rem_decode"][i]
            call.ready_since = cols["ready_since"][i]
            call.preemptions = cols["preempt"][i]
            sess.append(call)
            pol.register_call(call)
            f = cols["flags"][i]
            if f & F_ACTIVE:
                active[sid] = call
                lv = cols["level"][i]
                if self.mars:
                    pol.states[sid] = PriorityState(
                        level=lv, base_level=lv, served_tokens_at_level=cols["served"][i],
                        wait_since=cols["wait_since"][i], promotions=cols["promos"][i])
                else:
                    call.served_tokens = cols["served"][i]
            if f & F_PINNED:
                call.pinned = True
                call.retention_deadline = cols["deadline"][i]
                pb = cols["pinned_blocks"][i]
                pool.pinned[sid] = pb
                used += pb
                pol.pinned[sid] = PinnedSession(sid, pb, 0.0, 0.0, cols["deadline"][i],
                                                cols["plevel"][i] if self.mars else 0)
            elif call.kv_tokens > 0:
                h = A.blocks_for_tokens(call.kv_tokens, 16)
                pool.allocated[sid] = h
                used += h
            if f & F_BOUNDARY:
                boundary.append(call)
        pool.free_blocks = snap.total_blocks - used
        if pool.free_blocks != snap.free_blocks:
            raise ValueError("snapshot free_blocks inconsistent with its rows")
        self.queue = [A.QueueEntry(call=sess[r], req_blocks=cols["req_blocks"][r],
                                   is_long_session=bool(cols["flags"][r] & F_LONG),
                                   enqueue_time=0.0)
                      for r in snap.queue.tolist()]
        self.pol, self.pool, self.tel = pol, pool, tel
        self.sess, self.active, self.boundary = sess, active, boundary

    def run(self) -> dict:
        """The timed part: one scheduling step; returns small counters."""
        if self.port is not None:
            from oracle.snapshot_step import run_step
            out = run_step(self.snap, control_due=self.control_due, world=self.port)
            return {"window": len(out["window"]), "evictions": len(out["evictions"])}
        A = self.A
        from agentsched.scheduler import RetentionConfig, decide_retention
        from agentsched.telemetry import refresh_pressure

        snap, pol, pool, tel, now = self.snap, self.pol, self.pool, self.tel, self.snap.now
        active = self.active

        def evict(sid, kind):  # sim.py:168-188
            call = pol.calls[sid]
            if kind == "pinned":
                pool.release_pinned(sid)
                call.pinned = False
                call.retention_deadline = None
            else:
                pool.free(sid)
            call.kv_tokens = 0
            if kind == "running":
                call.preemptions += 1
                if call.phase == A.Phase.DECODE:
                    call.set_phase(A.Phase.PREFILL)
            pol.on_evicted(sid)

        for sid in pol.expired_pins(now):
            evict(sid, "pinned")

        class Plane:
            worker_slots = snap.worker_slots

            def active_count(self):
                return snap.active_tools

            def queued_count(self):
                return snap.queued_tools

        tel.probe(pool, Plane(), active_sessions=len(active))
        admitted = []
        if self.control_due:
            refresh_pressure(tel, self.pressure, snap.worker_slots)
            clock = A.SimClock()
            clock.now = now
            admitted = A.balance_and_admit(self.queue, self.ctl, tel, snap.worker_slots,
                                           self.pressure, clock, A.EventLog())
            for e in admitted:
                call = e.call
                call.admit_time = now
                A.submit_round(call, now)
                tel.record("gpu_submit", {"projected_blocks": call.incremental_blocks(
                    call.remaining_prefill, pool.block_size)})
                active[call.session_id] = call
                pol.on_admit(call, now)
        rc = RetentionConfig()
        for call in self.boundary:
            if self.mars:
                decide_retention(call, tel, pool, self.gpu, rc, self.pressure, now)
            else:
                pol.retention_decision(call, pool, tel, self.gpu, now)
        ready = [x for x in active.values() if x.phase in (A.Phase.PREFILL, A.Phase.DECODE)]
        ready.sort(key=lambda x: x.session_id)  # sim.py:339-340
        plan = pol.plan_tick(ready, pool, self.gpu, tel, now,
                             lambda v: evict(v.session_id, v.kind)) if ready else None
        return {"admitted": len(admitted), "ready": len(ready),
                "evictions": len(plan.evictions) if plan else 0,
                "tokens": plan.total_tokens if plan else 0}


def timed_step(snap, control_due: bool = True, policy: str = "mars") -> float:
    """Materialise (untimed), then time one step; seconds."""
    import time

    r = RefStep(snap, control_due=control_due, policy=policy)
    t0 = time.perf_counter()
    r.run()
    return time.perf_counter() - t0
