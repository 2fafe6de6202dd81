"""Oracle data-plane mechanisms and the MARS policy composition.

Restates ``agentsched/scheduler.py`` (MLFQ levels, quotas, aging, chunk
fitting, retention economics, reclamation order, plan builder) and
``agentsched/baselines.py:MarsPolicy``; TEST INFRASTRUCTURE ONLY.
"""

from __future__ import annotations

import math
from typing import Callable, Dict, List, Optional, Sequence, Tuple

from .core import DECODE, PREFILL, BlockCounter, ContractViolation, Session, TickModel, ceil_div
from .admission import Counters, Pressure

# scheduler.py:34-41
LEVELS = 4
BOUNDS = (4_000, 32_000, 128_000, math.inf)
QUOTAS = (2_000, 8_000, 32_000, math.inf)
AGING_S = 10.0
DECODE_SLOTS = 64
SLACK = 2.0
HORIZON_S = 60.0
PW_CLIP = 100.0


class Mlfq:
    """MlfqConfig (scheduler.py:44-63)."""

    def __init__(self, num_levels=LEVELS, level_boundaries_tokens=BOUNDS,
                 level_quotas_tokens=QUOTAS, promotion_wait_s=AGING_S,
                 max_promotions=LEVELS - 1, max_decode_slots=DECODE_SLOTS) -> None:
        self.num_levels = num_levels
        self.level_boundaries_tokens = tuple(level_boundaries_tokens)
        self.level_quotas_tokens = tuple(level_quotas_tokens)
        self.promotion_wait_s = promotion_wait_s
        self.max_promotions = max_promotions
        self.max_decode_slots = max_decode_slots

    @property
    def window_size(self) -> int:
        return 2 * self.max_decode_slots


class Retention:
    """RetentionConfig (scheduler.py:66-70)."""

    def __init__(self, deadline_slack=SLACK, max_pin_horizon_s=HORIZON_S,
                 pressure_weight_clip=PW_CLIP) -> None:
        self.deadline_slack = deadline_slack
        self.max_pin_horizon_s = max_pin_horizon_s
        self.pressure_weight_clip = pressure_weight_clip


class Prio:
    """PriorityState (scheduler.py:78-84)."""

    __slots__ = ("level", "base_level", "served_tokens_at_level", "wait_since", "promotions")

    def __init__(self, level: int, base_level: int, served: int = 0,
                 wait_since: float = 0.0, promotions: int = 0) -> None:
        self.level = level
        self.base_level = base_level
        self.served_tokens_at_level = served
        self.wait_since = wait_since
        self.promotions = promotions


def level_for(tokens: int, m: Mlfq) -> int:  # scheduler.py:87-97
    if tokens < 1:
        raise ContractViolation("context_tokens must be >= 1")
    for i, b in enumerate(m.level_boundaries_tokens):
        if tokens <= b:
            return i
    return m.num_levels - 1


def charge(st: Prio, tokens: int, m: Mlfq) -> None:  # scheduler.py:100-108
    if tokens < 0:
        raise ContractViolation("cannot charge negative service")
    st.served_tokens_at_level += tokens
    if st.served_tokens_at_level > m.level_quotas_tokens[st.level] and st.level < m.num_levels - 1:
        st.level += 1
        st.served_tokens_at_level = 0


def age(states, now: float, m: Mlfq) -> List[Prio]:  # scheduler.py:111-128
    moved = []
    for st in states:
        if st.level == 0 or st.promotions >= m.max_promotions:
            continue
        if now - st.wait_since >= m.promotion_wait_s:
            st.level -= 1
            st.promotions += 1
            st.wait_since = now
            moved.append(st)
    return moved


def fit_chunk(s: Session, desired: int, pool: BlockCounter, bs: int) -> int:
    """try_fit (scheduler.py:136-157)."""
    if desired < 1:
        raise ContractViolation("desired_tokens must be >= 1")
    held = ceil_div(s.kv_tokens, bs)
    room = (held + pool.free_blocks) * bs - s.kv_tokens
    grant = desired if desired <= room else (room // bs) * bs
    if grant < 1:
        return 0
    need = s.incremental_blocks(grant, bs)
    if need > 0 and not pool.allocate(s.session_id, need):
        raise ContractViolation("try_fit sized a grant the pool refused")
    return grant


class Pin:
    """PinnedSession (scheduler.py:165-172)."""

    __slots__ = ("session_id", "pinned_blocks", "pinned_at", "predicted_return",
                 "retention_deadline", "level")

    def __init__(self, session_id, pinned_blocks, pinned_at, predicted_return,
                 retention_deadline, level) -> None:
        self.session_id = session_id
        self.pinned_blocks = pinned_blocks
        self.pinned_at = pinned_at
        self.predicted_return = predicted_return
        self.retention_deadline = retention_deadline
        self.level = level


class Decision:
    """RetentionDecision (scheduler.py:175-180)."""

    __slots__ = ("pin", "benefit_s", "cost_s", "retention_deadline")

    def __init__(self, pin: bool, benefit_s: float, cost_s: float, retention_deadline: float):
        self.pin = pin
        self.benefit_s = benefit_s
        self.cost_s = cost_s
        self.retention_deadline = retention_deadline


def pressure_weight(u: float, clip: float = PW_CLIP) -> float:  # scheduler.py:183-187
    return clip if u >= 1.0 else min(1.0 / (1.0 - u), clip)


def retention(s: Session, t: Counters, pool: BlockCounter, gpu: TickModel,
              rc: Retention, p: Pressure, now: float) -> Decision:
    """decide_retention (scheduler.py:190-213); operation order kept exactly."""
    ema = t.effective_tool_estimate(p)
    benefit = s.context_tokens / gpu.prefill_rate
    foot = s.held_blocks(pool.block_size)
    cost = (foot / pool.total_blocks) * ema * pressure_weight(t.kv_usage_ratio, rc.pressure_weight_clip)
    pin = benefit > cost and ema <= rc.max_pin_horizon_s
    deadline = now + min(ema * rc.deadline_slack, rc.max_pin_horizon_s)
    return Decision(pin, benefit, cost, deadline)


class Victim:
    """scheduler.py:221-225."""

    __slots__ = ("session_id", "kind", "blocks")

    def __init__(self, session_id: str, kind: str, blocks: int) -> None:
        self.session_id = session_id
        self.kind = kind
        self.blocks = blocks

    def as_tuple(self):
        return (self.session_id, self.kind, self.blocks)


def choose_victims(need: int, pool: BlockCounter, pins: Dict[str, Pin],
                   running: Sequence[Session], level_of: Callable[[Session], int],
                   now: float) -> List[Victim]:
    """reclaim_for (scheduler.py:228-267)."""
    if need < 1:
        raise ContractViolation("needed_blocks must be >= 1")
    if pool.free_blocks >= need:
        return []
    cands = []
    for ps in pins.values():
        cands.append(((0 if ps.retention_deadline < now else 1, -ps.level, -ps.pinned_blocks,
                       ps.session_id), Victim(ps.session_id, "pinned", ps.pinned_blocks)))
    for s in running:
        h = s.held_blocks(pool.block_size)
        if h:
            cands.append(((2, -level_of(s), -h, s.session_id), Victim(s.session_id, "running", h)))
    cands.sort(key=lambda kv: kv[0])
    out: List[Victim] = []
    got = 0
    for _, v in cands:
        out.append(v)
        got += v.blocks
        if pool.free_blocks + got >= need:
            return out
    return []


class Plan:
    """TickPlan (scheduler.py:275-280)."""

    def __init__(self) -> None:
        self.decode_ids: List[str] = []
        self.prefill_grants: List[Tuple[str, int]] = []
        self.evictions: List[Victim] = []
        self.total_tokens = 0


def make_plan(ready: Sequence[Session], pool: BlockCounter, gpu: TickModel,
              key: Callable[[Session], tuple], window_size: int, decode_slots: int,
              shrink: bool, reclaimer, evict, strict_order: bool = False,
              window_out: Optional[list] = None) -> Plan:
    """build_plan (scheduler.py:283-371)."""
    plan = Plan()
    budget = gpu.token_budget_per_tick
    bs = pool.block_size
    window = sorted(ready, key=key)[:window_size]
    if window_out is not None:
        window_out.extend(window)
    planned: List[str] = []

    def claim(need: int, who: Session) -> bool:
        if pool.free_blocks >= need:
            return True
        if reclaimer is None or evict is None:
            return False
        vs = reclaimer(need, who, planned)
        if not vs:
            return False
        for v in vs:
            evict(v)
            plan.evictions.append(v)
        return pool.free_blocks >= need

    ndec = 0
    for s in window:
        if s.phase != DECODE or s.remaining_decode < 1:
            continue
        if plan.total_tokens >= budget or ndec >= decode_slots:
            continue
        need = s.incremental_blocks(1, bs)
        if need > 0:
            if not claim(need, s):
                continue
            if not pool.allocate(s.session_id, need):
                continue
        plan.decode_ids.append(s.session_id)
        planned.append(s.session_id)
        plan.total_tokens += 1
        ndec += 1

    for s in window:
        if s.phase != PREFILL:
            continue
        left = budget - plan.total_tokens
        if left < 1:
            break
        want = min(s.remaining_prefill, left)
        if want < 1:
            continue
        if shrink:
            g = fit_chunk(s, want, pool, bs)
            if g == 0 and claim(s.incremental_blocks(want, bs), s):
                g = fit_chunk(s, want, pool, bs)
        else:
            need = s.incremental_blocks(want, bs)
            if need == 0:
                g = want
            elif claim(need, s) and pool.allocate(s.session_id, need):
                g = want
            else:
                g = 0
        if g > 0:
            plan.prefill_grants.append((s.session_id, g))
            planned.append(s.session_id)
            plan.total_tokens += g
        elif strict_order:
            break
    return plan


# ---------------------------------------------------------------------------
# MARS policy (baselines.py:318-455)
# ---------------------------------------------------------------------------


class MarsOracle:
    """Hook surface of ``PolicyBase`` (baselines.py:56-101) with MarsPolicy's rules."""

    name = "mars"
    uses_admission_control = True

    def __init__(self, mlfq: Optional[Mlfq] = None, ret: Optional[Retention] = None,
                 pressure: Optional[Pressure] = None, enable_coordinator: bool = True,
                 enable_coscheduler: bool = True) -> None:
        self.mlfq = mlfq or Mlfq()
        self.retention = ret or Retention()
        self.pressure = pressure or Pressure()
        self.enable_coordinator = enable_coordinator
        self.enable_coscheduler = enable_coscheduler
        self.calls: Dict[str, Session] = {}
        self.states: Dict[str, Prio] = {}
        self.pinned: Dict[str, Pin] = {}
        self.last_window: List[Session] = []

    def register_call(self, call) -> None:
        self.calls[call.session_id] = call

    def on_admit(self, call, now: float) -> None:
        lv = level_for(call.rounds[0].new_prefill_tokens, self.mlfq)
        self.states[call.session_id] = Prio(lv, lv, wait_since=now)

    def on_resume(self, call, now: float) -> None:
        st = self.states.get(call.session_id)
        if st is not None:
            st.wait_since = now

    def on_service(self, sid: str, tokens: int, now: float) -> None:
        st = self.states.get(sid)
        if st is None or not self.enable_coordinator:
            return
        charge(st, tokens, self.mlfq)
        st.wait_since = now

    def level_of(self, call) -> int:
        return self.states[call.session_id].level if self.enable_coordinator else 0

    def order_key(self, call) -> tuple:
        if not self.enable_coordinator:
            return (call.arrival_time, call.session_id)
        return (self.states[call.session_id].level, call.ready_since, call.session_id)

    def retention_decision(self, call, pool, telemetry, gpu, now):
        if not self.enable_coscheduler:
            return None
        return retention(call, telemetry, pool, gpu, self.retention, self.pressure, now)

    def note_pin(self, call, decision, blocks: int, now: float) -> None:
        self.pinned[call.session_id] = Pin(call.session_id, blocks, now,
                                           now + self.pressure.initial_tool_estimate_s,
                                           decision.retention_deadline, self.level_of(call))

    def expired_pins(self, now: float) -> List[str]:
        return sorted(sid for sid, ps in self.pinned.items() if ps.retention_deadline < now)

    def on_evicted(self, sid: str) -> None:
        self.pinned.pop(sid, None)

    def _reclaimer(self, ready: Sequence[Session], now: float, pool: BlockCounter):
        def pick(need: int, who, planned: Sequence[str]) -> List[Victim]:
            bs = pool.block_size
            if self.enable_coordinator:
                mine = (self.level_of(who), who.ready_since, who.session_id)
                run = [c for c in ready
                       if c.session_id != who.session_id and c.session_id not in planned
                       and c.held_blocks(bs) > 0
                       and (self.level_of(c), c.ready_since, c.session_id) > mine]
                return choose_victims(need, pool, self.pinned, run, self.level_of, now)
            run = [c for c in ready
                   if c.session_id != who.session_id and c.session_id not in planned
                   and c.arrival_time > who.arrival_time and c.held_blocks(bs) > 0]
            return choose_victims(need, pool, self.pinned, run, lambda c: 0, now)
        return pick

    def plan_tick(self, ready, pool, gpu, telemetry, now, evictor) -> Plan:
        if self.enable_coordinator:
            age([self.states[c.session_id] for c in ready], now, self.mlfq)
        self.last_window = []
        return make_plan(ready, pool, gpu, self.order_key, self.mlfq.window_size,
                         self.mlfq.max_decode_slots, self.enable_coscheduler,
                         self._reclaimer(ready, now, pool), evictor,
                         window_out=self.last_window)


# ---------------------------------------------------------------------------
# Comparison policies (baselines.py:104-315) sharing the same plan builder
# ---------------------------------------------------------------------------

K_STATIC_TTL_S = 30.0          # baselines.py:50
K_DYNAMIC_TTL_MULTIPLIER = 1.5  # baselines.py:51


def arrival_key(s) -> tuple:  # baselines.py:104-105
    return (s.arrival_time, s.session_id)


def _prefix_victims(cands: Sequence[Session], need: int, pool: BlockCounter,
                    chosen: Optional[List[Victim]] = None, freed: int = 0) -> List[Victim]:
    """Shortest prefix of running candidates whose blocks cover the shortfall,
    else [] (baselines.py:129-138)."""
    chosen = list(chosen or [])
    for c in cands:
        b = c.held_blocks(pool.block_size)
        chosen.append(Victim(c.session_id, "running", b))
        freed += b
        if pool.free_blocks + freed >= need:
            return chosen
    return []


class _BaselineOracle:
    """PolicyBase defaults (baselines.py:56-101): no admission control, no pins."""

    name = "base"
    uses_admission_control = False
    strict_order = False

    def __init__(self, window_size: int = 128, max_decode_slots: int = DECODE_SLOTS) -> None:
        self.window_size = window_size
        self.max_decode_slots = max_decode_slots
        self.calls: Dict[str, Session] = {}
        self.last_window: List[Session] = []

    def register_call(self, call) -> None:
        self.calls[call.session_id] = call

    def on_admit(self, call, now: float) -> None:
        pass

    def on_resume(self, call, now: float) -> None:
        pass

    def on_service(self, sid: str, tokens: int, now: float) -> None:
        pass

    def retention_decision(self, call, pool, telemetry, gpu, now):
        return None

    def note_pin(self, call, decision, blocks: int, now: float) -> None:
        pass

    def expired_pins(self, now: float) -> List[str]:
        return []

    def on_evicted(self, sid: str) -> None:
        pass

    def order_key(self, call) -> tuple:
        return arrival_key(call)

    def _running(self, ready, who, planned, bs):
        raise NotImplementedError

    def _reclaimer(self, ready: Sequence[Session], now: float, pool: BlockCounter):
        def pick(need: int, who, planned: Sequence[str]) -> List[Victim]:
            return _prefix_victims(self._running(ready, who, planned, pool.block_size), need, pool)
        return pick

    def plan_tick(self, ready, pool, gpu, telemetry, now, evictor) -> Plan:
        self.last_window = []
        return make_plan(ready, pool, gpu, self.order_key, self.window_size,
                         self.max_decode_slots, False, self._reclaimer(ready, now, pool), evictor,
                         strict_order=self.strict_order, window_out=self.last_window)


class FcfsOracle(_BaselineOracle):
    """FcfsPolicy (baselines.py:108-155): arrival order, head-of-line blocking,
    victims are later arrivals, latest first."""

    name = "fcfs"
    strict_order = True

    def _running(self, ready, who, planned, bs):
        c = [s for s in ready if s.session_id != who.session_id and s.session_id not in planned
             and s.arrival_time > who.arrival_time and s.held_blocks(bs) > 0]
        c.sort(key=lambda s: (-s.arrival_time, s.session_id))
        return c


class ProgramPriorityOracle(_BaselineOracle):
    """ProgramPriorityPolicy (baselines.py:158-208): least cumulative service
    first; victims have more service, most first."""

    name = "program_priority"

    def order_key(self, call) -> tuple:
        return (call.served_tokens, call.arrival_time, call.session_id)

    def _running(self, ready, who, planned, bs):
        c = [s for s in ready if s.session_id != who.session_id and s.session_id not in planned
             and s.served_tokens > who.served_tokens and s.held_blocks(bs) > 0]
        c.sort(key=lambda s: (-s.served_tokens, s.session_id))
        return c


class TtlOracle(_BaselineOracle):
    """TtlPolicy (baselines.py:211-315): fcfs order plus unconditional pins
    with a static or EMA-scaled deadline; pins are reclaimed first (expired,
    then earliest deadline, then largest), then later arrivals."""

    strict_order = True

    def __init__(self, kind: str, pressure: Optional[Pressure] = None,
                 ttl_seconds: float = K_STATIC_TTL_S, multiplier: float = K_DYNAMIC_TTL_MULTIPLIER,
                 window_size: int = 128, max_decode_slots: int = DECODE_SLOTS) -> None:
        super().__init__(window_size, max_decode_slots)
        if kind not in ("static_ttl", "dynamic_ttl"):
            raise ValueError(kind)
        self.name = kind
        self.pressure = pressure or Pressure()
        self.ttl_seconds = ttl_seconds
        self.multiplier = multiplier
        self.pinned: Dict[str, Pin] = {}

    def retention_decision(self, call, pool, telemetry, gpu, now):
        if self.name == "static_ttl":
            deadline = now + self.ttl_seconds
        else:
            deadline = now + self.multiplier * telemetry.effective_tool_estimate(self.pressure)
        return Decision(True, 0.0, 0.0, deadline)

    def note_pin(self, call, decision, blocks: int, now: float) -> None:
        self.pinned[call.session_id] = Pin(call.session_id, blocks, now,
                                           decision.retention_deadline,
                                           decision.retention_deadline, 0)

    def expired_pins(self, now: float) -> List[str]:
        return sorted(sid for sid, ps in self.pinned.items() if ps.retention_deadline < now)

    def on_evicted(self, sid: str) -> None:
        self.pinned.pop(sid, None)

    def _reclaimer(self, ready: Sequence[Session], now: float, pool: BlockCounter):
        def pick(need: int, who, planned: Sequence[str]) -> List[Victim]:
            chosen: List[Victim] = []
            freed = 0
            pins = sorted(self.pinned.values(),
                          key=lambda ps: (0 if ps.retention_deadline < now else 1,
                                          ps.retention_deadline, -ps.pinned_blocks, ps.session_id))
            for ps in pins:
                chosen.append(Victim(ps.session_id, "pinned", ps.pinned_blocks))
                freed += ps.pinned_blocks
                if pool.free_blocks + freed >= need:
                    return chosen
            run = [s for s in ready if s.session_id != who.session_id
                   and s.session_id not in planned and s.arrival_time > who.arrival_time
                   and s.held_blocks(pool.block_size) > 0]
            run.sort(key=lambda s: (-s.arrival_time, s.session_id))
            return _prefix_victims(run, need, pool, chosen, freed)
        return pick


def make_oracle_policy(kind: str, **kw):
    """make_policy (baselines.py:458-495) over the oracle policies."""
    if kind == "mars":
        return MarsOracle(**kw)
    if kind == "fcfs":
        return FcfsOracle(**kw)
    if kind == "program_priority":
        return ProgramPriorityOracle(**kw)
    if kind in ("static_ttl", "dynamic_ttl"):
        return TtlOracle(kind, **kw)
    raise ValueError(kind)
