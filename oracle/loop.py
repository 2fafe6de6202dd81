"""Oracle tick loop: arrivals, tool returns, pin expiry, probe, control
cadence, plan, GPU tick, round completion.

Restates ``agentsched/sim.py:run_simulation`` so that tests on the GPU box
(where ``/root/reference`` does not exist) can drive any policy object --
the oracle's or the B200 drop-in -- through the reference's exact tick order
and compare the resulting event log byte for byte against the frozen
reference logs in ``tests/golden/``.  TEST INFRASTRUCTURE ONLY.
"""

from __future__ import annotations

import math
from typing import Dict, List, Optional, Sequence, Set, Tuple

from . import admission as adm
from .core import (BLOCK, CONTEXT_LIMIT, DECODE, DONE, PREFILL, TICK_S, TOKEN_BUDGET, TOOL,
                   WAITING_RESUME, BlockCounter, Clock, ContractViolation, Journal, Round,
                   Session, TickModel, ToolSlots, ceil_div, execute_tick, resume_cost,
                   submit_round)
from .tracefile import Trace

MAX_TICKS = 2_000_000


class Stall(RuntimeError):
    """SimulationStall (sim.py:56-57)."""


class Engine:
    """EngineParams (sim.py:60-74)."""

    def __init__(self, total_blocks: int, block_size: int = BLOCK,
                 token_budget_per_tick: int = TOKEN_BUDGET, tick_duration_s: float = TICK_S,
                 context_limit_tokens: int = CONTEXT_LIMIT, tool_worker_slots: int = 8) -> None:
        self.total_blocks = total_blocks
        self.block_size = block_size
        self.token_budget_per_tick = token_budget_per_tick
        self.tick_duration_s = tick_duration_s
        self.context_limit_tokens = context_limit_tokens
        self.tool_worker_slots = tool_worker_slots

    def gpu(self) -> TickModel:
        return TickModel(self.token_budget_per_tick, self.tick_duration_s, self.context_limit_tokens)



class RunOut:
    def __init__(self, log: Journal, calls: Dict[str, Session], counters: Dict[str, int],
                 horizon: float, pool: BlockCounter) -> None:
        self.log = log
        self.events = log.records
        self.calls = calls
        self.counters = counters
        self.horizon_s = horizon
        self.pool = pool


class _Empty:
    decode_ids: List[str] = []
    prefill_grants: List[Tuple[str, int]] = []
    evictions: list = []
    total_tokens = 0


def run(traces: Sequence[Trace], eng: Engine, policy, controller: Optional[adm.Controller] = None,
        pressure: Optional[adm.Pressure] = None, enable_control_plane: bool = True,
        max_ticks: int = MAX_TICKS, session_factory=Session, round_factory=Round,
        on_tick=None, balance_and_admit=None) -> RunOut:
    """One deterministic run.  ``policy`` is any object with the PolicyBase
    hooks (baselines.py:56-101); ``balance_and_admit`` any function with the
    reference signature (control.py:166-174), default the oracle's."""
    if balance_and_admit is None:
        def balance_and_admit(q, st, tel, slots, p, clk, lg):
            return adm.admit_step(q, st, tel, slots, p, clk.now, lg)
    ctl = controller or adm.Controller()
    prs = pressure or adm.Pressure()
    gpu = eng.gpu()
    for tr in traces:  # sim.py:103-109
        if ceil_div(tr.total_context_tokens, eng.block_size) > eng.total_blocks:
            raise ContractViolation(f"session {tr.session_id} cannot fit the pool")
    pool = BlockCounter(eng.total_blocks, eng.block_size)
    tools = ToolSlots(eng.tool_worker_slots)
    clock = Clock()
    log = Journal()
    tel = adm.Counters(pool.total_blocks)
    admission = enable_control_plane and policy.uses_admission_control

    def observe(op, sid, n, from_pinned):  # sim.py:118-124
        if from_pinned:
            log.emit(clock.now, op, sid, blocks=n, from_pinned=True)
        else:
            log.emit(clock.now, op, sid, blocks=n)

    pool.observer = observe

    def tel_emit(t, kind, sid, **payload):
        log.emit(t, kind, sid, **payload)
        tel.record(kind, payload, smoothing=prs.ema_smoothing)

    order = sorted(traces, key=lambda t: (t.arrival_time_s, t.session_id))
    nxt = 0
    queue: List[adm.Pending] = []
    active: Dict[str, Session] = {}
    first_seen: Set[Tuple[str, int]] = set()
    cnt = dict(admitted=0, completed=0, evictions=0, preemptions=0, warm_resumes=0,
               cold_resumes=0, pins=0, gpu_tokens=0)
    tick = gpu.tick_duration_s
    next_control = 0.0

    def admit(c: Session, now: float) -> None:  # sim.py:148-166
        c.admit_time = now
        submit_round(c, now)
        r = c.current_round()
        tel_emit(now, "gpu_submit", c.session_id, round=0, arrival_time=c.arrival_time,
                 required_prefill=c.remaining_prefill, new_tokens=r.new_prefill_tokens,
                 context_tokens=c.context_tokens, warm=None,
                 projected_blocks=c.incremental_blocks(c.remaining_prefill, pool.block_size))
        active[c.session_id] = c
        policy.on_admit(c, now)
        cnt["admitted"] += 1

    def evict(sid: str, kind: str, reason: str, t: float) -> None:  # sim.py:168-184
        c = policy.calls[sid]
        if kind == "pinned":
            n = pool.release_pinned(sid)
            c.pinned = False
            c.retention_deadline = None
        else:
            n = pool.free(sid)
        c.kv_tokens = 0
        if kind == "running":
            c.preemptions += 1
            cnt["preemptions"] += 1
            if c.phase == DECODE:
                c.set_phase(PREFILL)
        log.emit(t, "evict", sid, blocks=n, victim=kind, reason=reason)
        policy.on_evicted(sid)
        cnt["evictions"] += 1

    def plan_evict(v) -> None:  # sim.py:186-188
        evict(v.session_id, v.kind, "reclaim" if v.kind == "pinned" else "preempt", clock.now)

    def tool_return(c: Session, finish: float, now: float) -> None:  # sim.py:190-231
        c.round_index += 1
        c.set_phase(WAITING_RESUME)
        warm = c.pinned and c.retention_deadline is not None and c.retention_deadline >= finish
        need = resume_cost(c, warm)
        if warm:
            pool.unpin(c.session_id)
            c.pinned = False
            c.retention_deadline = None
            policy.on_evicted(c.session_id)
            c.warm_resumes += 1
            cnt["warm_resumes"] += 1
        else:
            if c.pinned:
                evict(c.session_id, "pinned", "pin_expired_at_return", now)
            c.cold_resumes += 1
            cnt["cold_resumes"] += 1
        new = c.current_round().new_prefill_tokens
        submit_round(c, now)
        if c.remaining_prefill != need:
            raise ContractViolation("resume cost mismatch")
        tel_emit(now, "gpu_submit", c.session_id, round=c.round_index, required_prefill=need,
                 new_tokens=new, context_tokens=c.context_tokens, warm=warm,
                 projected_blocks=c.incremental_blocks(need, pool.block_size))
        policy.on_resume(c, now)

    def round_done(c: Session, now: float) -> None:  # sim.py:233-279
        sid = c.session_id
        held = c.held_blocks(pool.block_size)
        tel.note_round_blocks(ceil_div(c.context_tokens, pool.block_size),
                              smoothing=prs.ema_smoothing)
        if c.is_last_round:
            c.completion_time = now
            c.set_phase(DONE)
            freed = pool.free(sid)
            c.kv_tokens = 0
            tel_emit(now, "gpu_end", sid, round=c.round_index, done=True, freed_blocks=freed)
            del active[sid]
            cnt["completed"] += 1
            return
        r = c.current_round()
        d = policy.retention_decision(c, pool, tel, gpu, now)
        if d is not None:
            log.emit(now, "retention", sid, pin=d.pin, benefit_s=d.benefit_s, cost_s=d.cost_s,
                     deadline=d.retention_deadline)
        if d is not None and d.pin and held > 0:
            pool.pin(sid)
            c.pinned = True
            c.retention_deadline = d.retention_deadline
            policy.note_pin(c, d, held, now)
            cnt["pins"] += 1
            freed = 0
        else:
            freed = pool.free(sid)
            c.kv_tokens = 0
            log.emit(now, "evict", sid, blocks=freed, victim="boundary", reason="tool_boundary")
            cnt["evictions"] += 1
        tel_emit(now, "gpu_end", sid, round=c.round_index, done=False, freed_blocks=freed)
        dur = r.tool_duration_s if r.tool_duration_s is not None else 0.0
        c.set_phase(TOOL)
        started = tools.start_tool(sid, dur, now)
        tel_emit(now, "tool_num", sid, queued=tools.queued_count(), duration_s=dur)
        if started:
            tel_emit(now, "tool_start", sid, duration_s=dur, active=tools.active_count())

    ticks = 0
    wedged = 0
    while nxt < len(order) or queue or active:  # sim.py:283-420
        if ticks > max_ticks:
            raise Stall(f"exceeded max_ticks={max_ticks}")
        ticks += 1
        now = clock.now
        while nxt < len(order) and order[nxt].arrival_time_s <= now + 1e-9:
            tr = order[nxt]
            nxt += 1
            c = session_factory(tr.session_id,
                                [round_factory(r.new_prefill_tokens, r.decode_tokens,
                                               r.tool_duration_s) for r in tr.rounds],
                                tr.arrival_time_s)
            policy.register_call(c)
            if admission:
                queue.append(adm.enqueue_entry(c, pool.total_blocks, pool.block_size, ctl, now))
            else:
                admit(c, now)
        done_tools = tools.complete_tools(now)
        for sid, start, dur in tools.take_promotions():
            tel_emit(start, "tool_start", sid, duration_s=dur, active=tools.active_count())
        for sid, start, fin, dur, qd in done_tools:
            tel_emit(fin, "tool_end", sid, duration_s=dur, queued_delay_s=qd)
            tool_return(policy.calls[sid], fin, now)
        for sid in policy.expired_pins(now):
            evict(sid, "pinned", "pin_expired", now)
        tel.probe(pool, tools, len(active))
        if admission and now >= next_control - 1e-9:
            adm.refresh_pressure(tel, prs, tools.worker_slots)
            log.emit(now, "telemetry", None, **tel.snapshot())
            for e in balance_and_admit(queue, ctl, tel, tools.worker_slots, prs, clock, log):
                admit(e.call, now)
            next_control = now + ctl.control_interval_s
        ready = [c for c in active.values() if c.phase in (PREFILL, DECODE)]
        ready.sort(key=lambda c: c.session_id)
        plan = policy.plan_tick(ready, pool, gpu, tel, now, plan_evict) if ready else _Empty()
        if on_tick is not None:
            on_tick(now, ready, plan)
        if plan.total_tokens > 0:
            wedged = 0
            log.emit(now, "tick", None, tokens=plan.total_tokens, decodes=list(plan.decode_ids),
                     prefills=[[sid, g] for sid, g in plan.prefill_grants],
                     evictions=len(plan.evictions))
            cnt["gpu_tokens"] += plan.total_tokens
            batch = [(policy.calls[sid], 0, True) for sid in plan.decode_ids]
            batch += [(policy.calls[sid], g, False) for sid, g in plan.prefill_grants]
            prog = execute_tick(clock, gpu, batch)
            end = clock.now
            for sid, pf, dd, pdone, rdone in prog:
                c = policy.calls[sid]
                policy.on_service(sid, pf + dd, end)
                if pdone and (sid, c.round_index) not in first_seen:
                    first_seen.add((sid, c.round_index))
                    tel_emit(end, "gpu_1st_token", sid, round=c.round_index,
                             launch_delay_s=end - c.round_submit_time)
                if rdone:
                    round_done(c, end)
            continue
        cands: List[float] = []
        if nxt < len(order):
            cands.append(order[nxt].arrival_time_s)
        nf = tools.next_finish_time()
        if nf is not None:
            cands.append(nf)
        if admission and (queue or active):
            cands.append(next_control)
        if ready or pool.pinned:
            cands.append(now + tick)
        busy = (tools.active_count() > 0 or tools.queued_count() > 0 or nxt < len(order)
                or bool(queue) or bool(pool.pinned))
        if ready and not busy:
            wedged += 1
            if wedged > math.ceil(len(ready) * 40.0 / tick) + 1024:
                raise Stall(f"{len(ready)} ready calls made no progress")
        else:
            wedged = 0
        if not cands:
            if active or queue:
                raise Stall("no future event but work remains")
            break
        target = min(cands)
        clock.advance(max(1, math.ceil((target - now) / tick - 1e-9)) * tick)
    log.emit(clock.now, "telemetry", None, **tel.snapshot())
    pool.check_conservation()
    return RunOut(log, dict(policy.calls), cnt, clock.now, pool)
