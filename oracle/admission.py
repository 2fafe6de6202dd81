"""Oracle control plane: telemetry counters/EMAs/overload hysteresis and the
external admission controller (queue packing, AIMD window, triple clamp).

Restates ``agentsched/telemetry.py`` and ``agentsched/control.py``;
TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).
"""

from __future__ import annotations

import math
from typing import List, Optional

from .core import ContractViolation, Session, ceil_div

# telemetry.py:14-19
EMA_ALPHA = 0.3
HYST = 3
CPU_HI, CPU_LO = 0.90, 0.70
KV_HI, KV_LO = 0.90, 0.70
TOOL_PRIOR_S = 5.0

# control.py:20-27
W_MIN = 2
AI = 1.0
MD = 0.5
CONTROL_S = 2.0
W_INIT = 8.0
CPU_OVERSUB = 1.5
RESERVE = 0.10
LONG_FRAC = 0.25

TELEMETRY_KINDS = ("gpu_submit", "gpu_1st_token", "gpu_end", "tool_num",
                   "tool_start", "tool_end", "window_update")


class Pressure:
    """PressureConfig (telemetry.py:38-56)."""

    def __init__(self, cpu_high_fraction=CPU_HI, cpu_low_fraction=CPU_LO,
                 kv_high_watermark=KV_HI, kv_low_watermark=KV_LO,
                 hysteresis_window=HYST, ema_smoothing=EMA_ALPHA,
                 initial_tool_estimate_s=TOOL_PRIOR_S) -> None:
        self.cpu_high_fraction = cpu_high_fraction
        self.cpu_low_fraction = cpu_low_fraction
        self.kv_high_watermark = kv_high_watermark
        self.kv_low_watermark = kv_low_watermark
        self.hysteresis_window = hysteresis_window
        self.ema_smoothing = ema_smoothing
        self.initial_tool_estimate_s = initial_tool_estimate_s


def ema_step(cur: float, x: float, a: float) -> float:  # telemetry.py:59-63
    if not (0 < a <= 1):
        raise ContractViolation("smoothing must be in (0, 1]")
    return a * x + (1.0 - a) * cur


class Counters:
    """The Telemetry value (telemetry.py:66-150, 152-166)."""

    def __init__(self, total_blocks: int) -> None:
        self.total_blocks = total_blocks
        self.available_kv = total_blocks
        self.kv_usage_ratio = 0.0
        self.active_tools = 0
        self.queued_tools = 0
        self.ema_tool_duration: Optional[float] = None
        self.ema_blocks_per_session: Optional[float] = None
        self.active_sessions = 0
        self.cpu_overloaded = False
        self.kv_overloaded = False
        self.last_window_update = 0.0
        self.last_w_adm: Optional[float] = None
        self.cpu_high_streak = 0
        self.cpu_low_streak = 0
        self.kv_high_streak = 0
        self.kv_low_streak = 0
        self.blocks_seed: Optional[float] = None

    def record(self, kind: str, payload: dict, smoothing: float = EMA_ALPHA) -> None:
        if kind not in TELEMETRY_KINDS:
            raise ContractViolation(f"unknown telemetry event kind {kind!r}")
        if kind == "tool_start":
            self.active_tools += 1
        elif kind == "tool_end":
            self.active_tools -= 1
            x = float(payload["duration_s"])
            self.ema_tool_duration = x if self.ema_tool_duration is None else ema_step(
                self.ema_tool_duration, x, smoothing)
        elif kind == "gpu_end":
            self.available_kv += int(payload["freed_blocks"])
        elif kind == "gpu_submit":
            self.available_kv -= int(payload["projected_blocks"])
        elif kind == "window_update":
            self.last_w_adm = float(payload["w_adm"])

    def effective_tool_estimate(self, p: Pressure) -> float:
        return p.initial_tool_estimate_s if self.ema_tool_duration is None else self.ema_tool_duration

    def note_round_blocks(self, blocks: int, smoothing: float = EMA_ALPHA) -> None:
        x = float(blocks)
        self.ema_blocks_per_session = x if self.ema_blocks_per_session is None else ema_step(
            self.ema_blocks_per_session, x, smoothing)

    def effective_blocks_per_session(self) -> float:
        if self.ema_blocks_per_session is not None:
            return self.ema_blocks_per_session
        if self.blocks_seed is not None:
            return self.blocks_seed
        return 1.0

    def probe(self, pool, tools, active_sessions: int) -> None:
        self.available_kv = pool.free_blocks
        self.kv_usage_ratio = pool.usage_ratio()
        self.active_tools = tools.active_count()
        self.queued_tools = tools.queued_count()
        self.active_sessions = active_sessions

    def snapshot(self) -> dict:
        return {
            "available_kv": self.available_kv,
            "kv_usage_ratio": self.kv_usage_ratio,
            "active_tools": self.active_tools,
            "queued_tools": self.queued_tools,
            "ema_tool_duration_s": self.ema_tool_duration,
            "ema_blocks_per_session": self.ema_blocks_per_session,
            "active_sessions": self.active_sessions,
            "cpu_overloaded": self.cpu_overloaded,
            "kv_overloaded": self.kv_overloaded,
        }


def _flip(on: bool, hi: bool, lo: bool, hs: int, ls: int, win: int):
    """One two-threshold hysteresis update; returns (on, hs, ls)."""
    hs = hs + 1 if hi else 0
    ls = ls + 1 if lo else 0
    if not on and hs >= win:
        return True, hs, 0
    if on and ls >= win:
        return False, 0, ls
    return on, hs, ls


def refresh_pressure(t: Counters, p: Pressure, worker_slots: int) -> None:
    """telemetry.py:174-208."""
    hi = t.active_tools >= p.cpu_high_fraction * worker_slots or t.queued_tools > 0
    lo = t.active_tools < p.cpu_low_fraction * worker_slots and t.queued_tools == 0
    t.cpu_overloaded, t.cpu_high_streak, t.cpu_low_streak = _flip(
        t.cpu_overloaded, hi, lo, t.cpu_high_streak, t.cpu_low_streak, p.hysteresis_window)
    hi = t.kv_usage_ratio >= p.kv_high_watermark
    lo = t.kv_usage_ratio < p.kv_low_watermark
    t.kv_overloaded, t.kv_high_streak, t.kv_low_streak = _flip(
        t.kv_overloaded, hi, lo, t.kv_high_streak, t.kv_low_streak, p.hysteresis_window)


def has_kv_slack(t: Counters, p: Pressure) -> bool:  # telemetry.py:211-213
    return t.kv_usage_ratio < p.kv_low_watermark


# ---------------------------------------------------------------------------
# Controller (control.py)
# ---------------------------------------------------------------------------


class Controller:
    """ControllerConfig (control.py:30-49) plus ControllerState (:52-61)."""

    def __init__(self, w_min=W_MIN, aimd_increase=AI, aimd_decrease=MD,
                 control_interval_s=CONTROL_S, initial_window=W_INIT,
                 cpu_oversubscription=CPU_OVERSUB, reserve_fraction=RESERVE,
                 long_session_fraction=LONG_FRAC) -> None:
        self.w_min = w_min
        self.aimd_increase = aimd_increase
        self.aimd_decrease = aimd_decrease
        self.control_interval_s = control_interval_s
        self.initial_window = initial_window
        self.cpu_oversubscription = cpu_oversubscription
        self.reserve_fraction = reserve_fraction
        self.long_session_fraction = long_session_fraction
        self.w_adm = float(initial_window)
        self.last_update = 0.0

    @property
    def config(self) -> "Controller":
        """ControllerState.config (control.py:56): the same object here."""
        return self


class Pending:
    """A queue entry (control.py:64-73)."""

    __slots__ = ("call", "req_blocks", "is_long_session", "enqueue_time")

    def __init__(self, call: Session, req_blocks: int, is_long_session: bool, enqueue_time: float):
        if req_blocks < 1:
            raise ContractViolation("queue entry needs req_blocks >= 1")
        self.call = call
        self.req_blocks = req_blocks
        self.is_long_session = is_long_session
        self.enqueue_time = enqueue_time


def enqueue_entry(call: Session, total_blocks: int, block: int, c: Controller, now: float) -> Pending:
    """control.py:76-93."""
    prefill = call.rounds[0].new_prefill_tokens
    if prefill < 1:
        raise ContractViolation("prefill_len must be >= 1")
    req = ceil_div(prefill, block)
    return Pending(call, req, req > c.long_session_fraction * total_blocks, now)


def pack(queue: List[Pending], t: Counters) -> List[Pending]:
    """control.py:101-122; stable, does not mutate ``queue``."""
    if t.cpu_overloaded:
        return sorted(queue, key=lambda e: -e.req_blocks)
    if queue and all(e.is_long_session for e in queue):
        cap = t.available_kv
        took, left = [], []
        for e in queue:
            if e.req_blocks <= cap:
                took.append(e)
                cap -= e.req_blocks
            else:
                left.append(e)
        return took + left
    return sorted(queue, key=lambda e: e.req_blocks)


def cpu_limit(t: Counters, worker_slots: int, c: Controller) -> float:  # control.py:130-132
    return max(float(c.w_min), worker_slots * c.cpu_oversubscription - t.queued_tools)


def kv_limit(t: Counters, c: Controller) -> float:  # control.py:135-138
    per = max(t.effective_blocks_per_session(), 1.0)
    cap = math.floor(t.available_kv * (1.0 - c.reserve_fraction) / per)
    return max(float(c.w_min), cap + t.active_sessions)


def window_limit(c: Controller, t: Counters, worker_slots: int, p: Pressure, now: float) -> int:
    """update_window (control.py:141-163)."""
    if now - c.last_update >= c.control_interval_s:
        if t.cpu_overloaded or t.kv_overloaded:
            c.w_adm = max(float(c.w_min), c.w_adm * c.aimd_decrease)
        elif has_kv_slack(t, p):
            c.w_adm = c.w_adm + c.aimd_increase
        c.last_update = now
    return int(min(c.w_adm, cpu_limit(t, worker_slots, c), kv_limit(t, c)))


def py_median(values: List[int]):
    """statistics.median: middle element, or the mean of the two middles."""
    s = sorted(values)
    n = len(s)
    if n == 0:
        raise ValueError("no median for empty data")
    if n % 2 == 1:
        return s[n // 2]
    return (s[n // 2 - 1] + s[n // 2]) / 2


def admit_step(queue: List[Pending], c: Controller, t: Counters, worker_slots: int,
               p: Pressure, now: float, log=None, stats: Optional[dict] = None) -> List[Pending]:
    """balance_and_admit (control.py:166-208): mutates ``queue`` in place.
    ``stats`` (optional) receives limit / slots / take."""
    if t.ema_blocks_per_session is None and t.blocks_seed is None and queue:
        t.blocks_seed = py_median([e.req_blocks for e in queue])
    order = pack(queue, t)
    limit = window_limit(c, t, worker_slots, p, now)
    slots = limit - t.active_sessions
    take = min(slots, len(order)) if slots > 0 else 0
    chosen = order[:take]
    queue[:] = order[take:]
    if stats is not None:
        stats.update(limit=limit, slots=slots, take=take)
    if log is not None:
        log.emit(now, "window_update", None, w_adm=c.w_adm, limit=limit, slots=slots,
                 admitted=[e.call.session_id for e in chosen],
                 cpu_overloaded=t.cpu_overloaded, kv_overloaded=t.kv_overloaded)
        t.record("window_update", {"w_adm": c.w_adm}, smoothing=p.ema_smoothing)
        t.last_window_update = now
    return chosen
