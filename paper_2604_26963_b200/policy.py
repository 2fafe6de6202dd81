"""``GpuMarsPolicy``: drop-in for ``agentsched.baselines.MarsPolicy``.

Same hook surface as the reference plugin API (``PolicyBase``,
baselines.py:56-101) and the same ablation switches (baselines.py:334-349);
register it under a new ``POLICY_KINDS`` entry or pass it to
``run_simulation`` directly.  Each ``plan_tick`` runs ONE device step on the
B200 (promote_waiting + window top-k + build_plan with chunk fitting and
reclamation, scheduler.py:111-128/283-371, baselines.py:406-455) and replays
the step's ordered journal through the caller's own ``KvPool`` and evictor, so
the reference's event log comes out byte-identical.

State ownership mirrors the reference: the sim owns ``Call`` objects and the
pool; the policy's MLFQ states and pin registry live in the device session
table.  ``charge_service`` (on_service) and ``decide_retention`` for rounds
that finish this tick are evaluated by the same device step, on post-tick
values (engine.py:503-512), and handed back when the sim asks for them.
"""

from __future__ import annotations

import ctypes as C
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .engine import MarsEngine, make_config
from .snapshot import COLUMNS, DECODE, F_ACTIVE, F_PINNED, PHASE_NAMES, PREFILL

ContractViolation = N.ContractViolation
_PHASE_CODE = {p: i for i, p in enumerate(PHASE_NAMES)}
_DROPIN_MODE = (N.MODE_SKIP_EXPIRY | N.MODE_SKIP_PROBE | N.MODE_SKIP_REFRESH | N.MODE_SERVICE
                | N.MODE_FINISH_RETENTION)


def _phase_code(phase) -> int:
    return _PHASE_CODE[getattr(phase, "value", phase)]


def _i64(x) -> int:
    return 2**63 - 1 if x == math.inf else int(x)


class _Victim:
    """scheduler.py:221-225 (fields read by the sim's evictor, sim.py:186-188)."""

    __slots__ = ("session_id", "kind", "blocks")

    def __init__(self, session_id: str, kind: str, blocks: int) -> None:
        self.session_id, self.kind, self.blocks = session_id, kind, blocks

    def __repr__(self) -> str:
        return f"Victim({self.session_id!r}, {self.kind!r}, {self.blocks})"


class _TickPlan:
    """scheduler.py:275-280."""

    def __init__(self) -> None:
        self.decode_ids: List[str] = []
        self.prefill_grants: List[Tuple[str, int]] = []
        self.evictions: List[Victim] = []
        self.total_tokens = 0


class _RetentionDecision:
    """scheduler.py:175-180."""

    __slots__ = ("pin", "benefit_s", "cost_s", "retention_deadline")

    def __init__(self, pin: bool, benefit_s: float, cost_s: float, retention_deadline: float):
        self.pin, self.benefit_s, self.cost_s = pin, benefit_s, cost_s
        self.retention_deadline = retention_deadline


# Inside the reference's own process (agentsched importable) the drop-ins ARE
# PolicyBase plugins and hand back the reference's plan / victim / decision
# types (baselines.py:56-101, scheduler.py:175-180, 221-225, 275-280);
# standalone they use the field-compatible classes above.
try:
    from agentsched.baselines import PolicyBase as _PolicyBase
    from agentsched.scheduler import RetentionDecision, TickPlan, Victim
except ImportError:  # the reference package is not installed
    _PolicyBase = object
    RetentionDecision, TickPlan, Victim = _RetentionDecision, _TickPlan, _Victim


def config_from(mlfq=None, retention=None, pressure=None, controller=None,
                enable_coordinator=True, enable_coscheduler=True, gpu=None,
                policy: str = "mars", **extra) -> N.MarsConfig:
    """mars_config from reference-style config objects (duck-typed)."""
    cfg = make_config(enable_coordinator, enable_coscheduler, policy=policy)
    for k, v in extra.items():
        setattr(cfg, k, v)
    if mlfq is not None:
        cfg.num_levels = mlfq.num_levels
        cfg.max_promotions = mlfq.max_promotions
        cfg.max_decode_slots = mlfq.max_decode_slots
        cfg.window_size = mlfq.window_size
        cfg.promotion_wait_s = float(mlfq.promotion_wait_s)
        for i in range(4):
            bs = list(mlfq.level_boundaries_tokens) + [math.inf] * 4
            qs = list(mlfq.level_quotas_tokens) + [math.inf] * 4
            cfg.level_bounds[i] = _i64(bs[i])
            cfg.level_quotas[i] = _i64(qs[i])
    if retention is not None:
        cfg.deadline_slack = float(retention.deadline_slack)
        cfg.max_pin_horizon_s = float(retention.max_pin_horizon_s)
        cfg.pressure_weight_clip = float(retention.pressure_weight_clip)
    if pressure is not None:
        for f in ("cpu_high_fraction", "cpu_low_fraction", "kv_high_watermark",
                  "kv_low_watermark", "ema_smoothing", "initial_tool_estimate_s"):
            setattr(cfg, f, float(getattr(pressure, f)))
        cfg.hysteresis_window = int(pressure.hysteresis_window)
    if controller is not None:
        cfg.w_min = int(controller.w_min)
        for f in ("aimd_increase", "aimd_decrease", "control_interval_s", "initial_window",
                  "cpu_oversubscription", "reserve_fraction", "long_session_fraction"):
            setattr(cfg, f, float(getattr(controller, f)))
    if gpu is not None:
        cfg.token_budget = int(gpu.token_budget_per_tick)
        cfg.tick_duration_s = float(gpu.tick_duration_s)
    return cfg


class GpuMarsPolicy(_PolicyBase):
    """B200 drop-in for MarsPolicy (baselines.py:318-455); a PolicyBase
    subclass whenever the reference package is importable.

    Device writes are batched: every hook records its row's new values on the
    host and the next plan_tick uploads them, one call per hook kind, in the
    order the hooks fire between two ticks (the previous tick's service
    charges and pins, then arrivals, tool returns, evictions, admissions), and
    only the ready rows whose Call changed since the last tick (new in the
    ready list, planned or evicted by the last plan, touched by a hook) are
    re-uploaded."""

    # hook kind -> the columns it sets, in the order hooks fire between ticks
    # (kinds with no columns run a device hook kernel: mars_on_service /
    # mars_on_admit, the reference's MLFQ arithmetic never restated on the host)
    _PENDING = (("service", ()), ("service_pre", ()),
                ("pin", ("flags", "deadline", "pinned_blocks", "plevel")),
                ("register", ("phase", "flags", "rank", "arrival")),
                ("resume", ("wait_since",)),
                ("evicted", ("flags", "kv")),
                ("admit", ()),
                ("admit_base", ("level", "promos", "served", "flags")))

    name = "mars"
    uses_admission_control = True
    # the drop-in step: no expiry / probe / refresh (the sim does those), MLFQ
    # charges at tick end and S2 for the rounds that finish this tick
    _mode = _DROPIN_MODE

    def __init__(self, mlfq=None, retention=None, pressure=None, enable_coordinator: bool = True,
                 enable_coscheduler: bool = True, max_sessions: int = 1 << 16,
                 device: int = 0, kv_blocks: bool = False) -> None:
        self._kv_enabled = kv_blocks
        self.kv = None                 # KvBlockManager once the pool is known
        self._kv_pending: List[tuple] = []
        self.mlfq, self.retention, self.pressure = mlfq, retention, pressure
        self.enable_coordinator = enable_coordinator
        self.enable_coscheduler = enable_coscheduler
        self._cfg_args = dict(mlfq=mlfq, retention=retention, pressure=pressure,
                              enable_coordinator=enable_coordinator,
                              enable_coscheduler=enable_coscheduler)
        self._max = int(max_sessions)
        self._device = device
        self.eng: Optional[MarsEngine] = None
        self._gpu_key = None
        self.calls: Dict[str, object] = {}
        self._row: Dict[str, int] = {}
        self._sid: List[str] = []
        self._max_sid: Optional[str] = None
        self._ranks_dirty = False
        self._pins: Dict[str, float] = {}       # sid -> retention deadline (registry view)
        self._levels: Dict[str, int] = {}       # sid -> MLFQ level (device value)
        self._admitted: set = set()
        self._fin: Dict[str, tuple] = {}        # sid -> (ctx, kv, now, usage, ema, decision)
        # sid -> (tokens, tick_end, level, served before the charge): charged on device
        self._service: Dict[str, tuple] = {}
        self._replaying = False
        self.last_window: List[str] = []
        self._tool_prior = getattr(pressure, "initial_tool_estimate_s", 5.0)
        self._pend: Dict[str, Dict[int, tuple]] = {k: {} for k, _ in self._PENDING}
        self._in_ready = np.zeros(self._max, bool)   # rows of the last uploaded ready list
        self._dirty = np.zeros(self._max, bool)      # rows whose Call changed since
        self._ready_rows = np.zeros(0, np.int64)

    # -- device context ---------------------------------------------------------

    def _engine(self, gpu=None) -> MarsEngine:
        if self.eng is None:
            cfg = config_from(gpu=gpu, **self._cfg_args)
            self._gpu_key = (cfg.token_budget, cfg.tick_duration_s)
            self.eng = MarsEngine(max_rows=self._max, max_queue=1, device=self._device,
                                  config=cfg)
            self.eng.set_graph(True)  # one CUDA-graph launch per plan_tick
        elif gpu is not None and (gpu.token_budget_per_tick, gpu.tick_duration_s) != self._gpu_key:
            # the sim registers and admits sessions before the first plan_tick
            # hands over the GpuModel (sim.py:165, :297, :342): the engine
            # parameters change in place, the registered rows stay
            self._gpu_key = (gpu.token_budget_per_tick, gpu.tick_duration_s)
            self.eng.set_config(config_from(gpu=gpu, **self._cfg_args))
        return self.eng

    def close(self) -> None:
        if self.eng is not None:
            self.eng.close()
            self.eng = None

    # -- PolicyBase hooks -----------------------------------------------------------

    def register_call(self, call) -> None:
        sid = call.session_id
        self.calls[sid] = call
        if sid in self._row:
            return
        if len(self._sid) >= self._max:
            raise RuntimeError(f"GpuMarsPolicy: more than max_sessions={self._max} sessions")
        r = len(self._sid)
        self._row[sid] = r
        # rank = position in lexicographic session-id order; a new id that is
        # not the largest so far shifts the ranks of every larger id
        if self._max_sid is not None and sid < self._max_sid:
            self._ranks_dirty = True
        else:
            self._max_sid = sid
        self._sid.append(sid)
        self._engine()
        self._queue("register", r, (_phase_code(call.phase), 0, r, call.arrival_time))
        # ranks only order the device step's keys: one re-rank in the next
        # plan_tick covers every out-of-order registration before it

    def _queue(self, kind: str, row: int, vals: tuple) -> None:
        self._pend[kind][row] = vals
        self._dirty[row] = True

    def _flush(self) -> None:
        """Uploads the hooks' pending row values (one call per hook kind)."""
        eng = None
        for kind, cols in self._PENDING:
            d = self._pend[kind]
            if not d:
                continue
            eng = eng or self._engine()
            rows = np.fromiter(d.keys(), np.int64, len(d))
            vals = list(zip(*d.values()))
            d.clear()
            P = C.c_void_p
            if kind == "admit":       # (first round's new prefill, now)
                r0 = np.asarray(vals[0], np.int32)
                now = np.asarray(vals[1], np.float64)
                eng._check(eng.lib.mars_on_admit(eng.ctx, len(rows), rows.ctypes.data_as(P),
                                                 r0.ctypes.data_as(P), now.ctypes.data_as(P)))
            elif kind in ("service", "service_pre"):   # (tokens, now[, pre-charge state])
                tok = np.asarray(vals[0], np.int64)
                now = np.asarray(vals[1], np.float64)
                pre = np.asarray(vals[2], np.int64) if kind == "service_pre" else None
                eng._check(eng.lib.mars_on_service(
                    eng.ctx, len(rows), rows.ctypes.data_as(P), tok.ctypes.data_as(P),
                    now.ctypes.data_as(P), pre.ctypes.data_as(P) if pre is not None else None))
            else:
                eng.upsert({c: np.asarray(v, dtype=COLUMNS[c]) for c, v in zip(cols, vals)},
                           rows=rows)

    def _sync_ranks(self) -> None:
        order = sorted(range(len(self._sid)), key=self._sid.__getitem__)
        rank = np.empty(len(order), np.uint32)
        rank[np.array(order, dtype=np.int64)] = np.arange(len(order), dtype=np.uint32)
        self._engine().upsert({"rank": rank}, rows=np.arange(len(order)))
        self._ranks_dirty = False

    def on_admit(self, call, now: float) -> None:
        sid = call.session_id
        tokens = call.rounds[0].new_prefill_tokens
        if tokens < 1:  # initial_level's precondition (scheduler.py:93-94)
            raise ContractViolation("context_tokens must be >= 1")
        # the level itself: initial_level on the device at the next upload
        self._queue("admit", self._row[sid], (tokens, now))
        self._admitted.add(sid)

    def on_resume(self, call, now: float) -> None:
        sid = call.session_id
        if sid in self._admitted:
            self._queue("resume", self._row[sid], (now,))

    def on_service(self, session_id: str, tokens: int, now: float) -> None:
        if session_id not in self._admitted or not self.enable_coordinator:
            return
        exp = self._service.pop(session_id, None)
        if exp is not None and exp[:2] == (tokens, now):
            return  # already charged by the device step at tick end
        if tokens < 0:  # charge_service's precondition (scheduler.py:102-103)
            raise ContractViolation("cannot charge negative service")
        r = self._row[session_id]
        if exp is not None:
            # the device charged its prediction: charge this amount from the
            # state before it instead (charge_service on the device)
            self._queue("service_pre", r, (int(tokens), now, (exp[3] << 8) | exp[2]))
        else:  # a charge the plan did not predict: from the device row's state
            self._queue("service", r, (int(tokens), now))

    def level_of(self, call) -> int:
        """The MLFQ level now (baselines.py:370-372): the device row, which
        the step's promote_waiting and charges keep current."""
        if not self.enable_coordinator:
            return 0
        r = self._row[call.session_id]
        self._flush()
        return int(self._engine().read(["level"], rows=np.array([r]))["level"][0])

    def retention_decision(self, call, pool, telemetry, gpu, now):
        if not self.enable_coscheduler:
            return None
        sid = call.session_id
        ema = telemetry.ema_tool_duration
        ema = self._tool_prior if ema is None else ema
        usage = telemetry.kv_usage_ratio
        pre = self._fin.pop(sid, None)
        if pre is not None and pre[:5] == (call.context_tokens, call.kv_tokens, now, usage, ema) \
                and pre[6] == pool.total_blocks:
            return pre[5]
        pin, b, c, d = self._engine().retention_batch(
            np.array([call.context_tokens]), np.array([call.kv_tokens]), pool.total_blocks,
            usage, ema, now)
        return RetentionDecision(bool(pin[0]), float(b[0]), float(c[0]), float(d[0]))

    def note_pin(self, call, decision, blocks: int, now: float) -> None:
        sid = call.session_id
        r = self._row[sid]
        # the round that ends here was planned this tick, so its post-charge
        # level came back with the step (no device read)
        lv = self._levels[sid] if self.enable_coordinator else 0
        self._queue("pin", r, (F_ACTIVE | F_PINNED, decision.retention_deadline, blocks, lv))
        self._pins[sid] = decision.retention_deadline

    def expired_pins(self, now: float) -> List[str]:
        """The pins whose deadline passed, in session-id order (baselines.py:
        396-399), found on the device from the table's pin flags and
        deadlines (the pending hook writes go up first)."""
        if not self._pins:
            return []
        self._flush()
        eng = self._engine()
        out = np.zeros(len(self._pins), np.uint32)
        n = C.c_int64()
        eng._check(eng.lib.mars_expired_pins(eng.ctx, float(now), len(out),
                                             out.ctypes.data_as(C.c_void_p), C.byref(n)))
        sid = self._sid
        return sorted(sid[r] for r in out[:n.value].tolist())

    def on_evicted(self, session_id: str) -> None:
        if self._pins.pop(session_id, None) is None:
            return
        if self._replaying:
            return  # the device step already released this pin
        r = self._row[session_id]
        call = self.calls[session_id]
        flags = F_ACTIVE if session_id in self._admitted else 0
        self._queue("evicted", r, (flags, call.kv_tokens))

    # -- the tick ---------------------------------------------------------------------

    def _extra_cols(self, calls: Sequence, n: int) -> dict:
        return {}

    # -- S5 block IDs: tee of the caller's pool op stream -------------------------

    def _kv_attach(self, pool, gpu) -> None:
        from .kvstore import OBSERVER_OPS, KvBlockManager

        per_row = -(-gpu.context_limit_tokens // pool.block_size) + 1
        self.kv = KvBlockManager(self._engine(gpu), pool.total_blocks,
                                 max_blocks_per_row=min(per_row, pool.total_blocks))
        inner = pool.observer

        def tee(op, sid, blocks, from_pinned=False):
            # ops the device step produced itself are already applied on the device
            if not self._replaying:
                self._kv_pending.append((OBSERVER_OPS[op], self._row[sid], int(blocks)))
            if inner is not None:
                inner(op, sid, blocks, from_pinned)

        pool.observer = tee

    def kv_flush(self) -> None:
        """Applies pool ops observed since the last step to the device tables."""
        if self.kv is not None and self._kv_pending:
            self.kv.apply(self._kv_pending)
            self._kv_pending = []

    def plan_tick(self, ready: Sequence, pool, gpu, telemetry, now: float, evictor) -> TickPlan:
        eng = self._engine(gpu)
        if self._kv_enabled and self.kv is None:
            self._kv_attach(pool, gpu)
        self.kv_flush()
        self._flush()
        if self._ranks_dirty:
            self._sync_ranks()
        rid = self._row
        rows = np.fromiter((rid[c.session_id] for c in ready), dtype=np.int64, count=len(ready))
        # re-upload only the ready rows whose Call can have changed: new in the
        # ready list, planned or evicted by the last plan, touched by a hook
        # (the sim changes a Call's phase / kv / context / decode / ready_since
        # only through those, engine.py:320-330, :459-514, sim.py:168-279)
        sel = np.nonzero(~self._in_ready[rows] | self._dirty[rows])[0]
        self._in_ready[self._ready_rows] = False
        self._in_ready[rows] = True
        gone = self._ready_rows[~self._in_ready[self._ready_rows]]
        self._ready_rows = rows
        n = len(sel)
        if n:
            calls = [ready[i] for i in sel.tolist()]
            cols = {
                "phase": np.fromiter((_phase_code(c.phase) for c in calls), np.uint8, n),
                "flags": np.full(n, F_ACTIVE, np.uint8),
                "kv": np.fromiter((c.kv_tokens for c in calls), np.int32, n),
                "context": np.fromiter((c.context_tokens for c in calls), np.int32, n),
                "rem_decode": np.fromiter((c.remaining_decode for c in calls), np.int32, n),
                "ready_since": np.fromiter((c.ready_since for c in calls), np.float64, n),
                "arrival": np.fromiter((c.arrival_time for c in calls), np.float64, n),
            }
            cols.update(self._extra_cols(calls, n))
            eng.upsert(cols, rows=rows[sel])
        if len(gone):
            eng.upsert({"phase": np.array([_phase_code(self.calls[self._sid[r]].phase)
                                           for r in gone.tolist()], np.uint8)}, rows=gone)
        self._dirty[:] = False
        s = N.MarsScalars()
        s.total_blocks = pool.total_blocks
        s.free_blocks = pool.free_blocks
        s.available_kv = pool.free_blocks
        s.kv_usage_ratio = float(telemetry.kv_usage_ratio)
        ema = telemetry.ema_tool_duration
        s.has_ema_tool = int(ema is not None)
        s.ema_tool = float(ema) if ema is not None else 0.0
        s.w_adm = 1.0
        eng.set_scalars(s)
        eng._check(eng.lib.mars_set_rows(eng.ctx, len(self._sid)))
        si = eng.step_in(now, False, 0, 0, 1, self._mode)
        res = eng.step(si)
        if res.status:
            raise RuntimeError(f"device step status {res.status}")
        # the plan's rows change in step_gpu / the evictor before the next tick
        self._dirty[res.decode_rows] = True
        self._dirty[res.prefill_rows] = True
        self._dirty[res.journal_row] = True
        sid = self._sid
        plan = TickPlan()
        self.last_window = [sid[r] for r in res.window_rows]
        # replay the ordered journal through the caller's pool and evictor so the
        # observer sees alloc / free / evict in build_plan's order
        self._replaying = True
        try:
            for op, r, k in zip(res.journal_op.tolist(), res.journal_row.tolist(),
                                res.journal_n.tolist()):
                if op == 1:
                    if not pool.allocate(sid[r], k):
                        raise ContractViolation(f"device plan allocation refused for {sid[r]}")
                else:
                    v = Victim(sid[r], "pinned" if op == 3 else "running", k)
                    evictor(v)
                    plan.evictions.append(v)
        finally:
            self._replaying = False
        plan.decode_ids = [sid[r] for r in res.decode_rows.tolist()]
        plan.prefill_grants = [(sid[r], int(g)) for r, g in zip(res.prefill_rows.tolist(),
                                                                 res.prefill_grants.tolist())]
        plan.total_tokens = int(res.total_tokens)
        tick_end = now + gpu.tick_duration_s
        self._service.clear()
        pre = res.plan_pre_charge.tolist()
        if not pre:
            pre = [0] * (len(res.decode_rows) + len(res.prefill_rows))
        nd = len(res.decode_rows)
        for i, (r, lv) in enumerate(zip(res.decode_rows.tolist(), res.decode_level.tolist())):
            self._levels[sid[r]] = lv
            self._service[sid[r]] = (1, tick_end, pre[i] & 0xff, pre[i] >> 8)
        for i, ((r, g), lv) in enumerate(zip(zip(res.prefill_rows.tolist(),
                                                 res.prefill_grants.tolist()),
                                             res.prefill_level.tolist())):
            self._levels[sid[r]] = lv
            self._service[sid[r]] = (g, tick_end, pre[nd + i] & 0xff, pre[nd + i] >> 8)
        self._fin.clear()
        ema_v = self._tool_prior if ema is None else ema
        for r, p, b, c, d in zip(res.fin_rows.tolist(), res.fin_pin.tolist(),
                                 res.fin_benefit.tolist(), res.fin_cost.tolist(),
                                 res.fin_deadline.tolist()):
            call = self.calls[sid[r]]
            self._fin[sid[r]] = (call.context_tokens + 1, call.kv_tokens + 1, tick_end,
                                 telemetry.kv_usage_ratio, ema_v,
                                 RetentionDecision(bool(p), b, c, d), pool.total_blocks)
        return plan


# ---------------------------------------------------------------------------
# The reference's comparison policies on the same device step
# ---------------------------------------------------------------------------


class _Slots:
    """The two MlfqConfig fields the comparison policies take (baselines.py:113-116)."""

    def __init__(self, window_size: int, max_decode_slots: int) -> None:
        self.window_size, self.max_decode_slots = window_size, max_decode_slots
        self.num_levels, self.max_promotions, self.promotion_wait_s = 4, 3, 10.0
        self.level_boundaries_tokens = (4_000, 32_000, 128_000, math.inf)
        self.level_quotas_tokens = (2_000, 8_000, 32_000, math.inf)


class _GpuComparisonPolicy(GpuMarsPolicy):
    """PolicyBase defaults (baselines.py:56-101) over the B200 step: no
    admission control, no MLFQ state, the window ordered by the policy's key
    and build_plan run with whole-chunk fitting (the device walk with
    mars_config.policy set).  The sim's pool and evictor see the same ordered
    journal replay as GpuMarsPolicy."""

    uses_admission_control = False
    _mode = N.MODE_SKIP_EXPIRY | N.MODE_SKIP_PROBE | N.MODE_SKIP_REFRESH

    def __init__(self, window_size: int = 128, max_decode_slots: int = 64,
                 max_sessions: int = 1 << 16, device: int = 0, kv_blocks: bool = False,
                 pressure=None, **cfg_extra) -> None:
        super().__init__(mlfq=_Slots(window_size, max_decode_slots), pressure=pressure,
                         enable_coordinator=False, enable_coscheduler=False,
                         max_sessions=max_sessions, device=device, kv_blocks=kv_blocks)
        self.window_size, self.max_decode_slots = window_size, max_decode_slots
        self._cfg_args.update(policy=self.name, **cfg_extra)

    def on_admit(self, call, now: float) -> None:
        r = self._row[call.session_id]
        self._engine().upsert({"level": np.zeros(1, np.uint8), "promos": np.zeros(1, np.uint8),
                               "served": np.array([call.served_tokens], np.int64),
                               "flags": np.array([F_ACTIVE], np.uint8)}, rows=np.array([r]))
        self._levels[call.session_id] = 0
        self._admitted.add(call.session_id)

    def on_resume(self, call, now: float) -> None:
        pass

    def on_service(self, session_id: str, tokens: int, now: float) -> None:
        pass

    def level_of(self, call) -> int:
        return 0

    def retention_decision(self, call, pool, telemetry, gpu, now):
        return None


class GpuFcfsPolicy(_GpuComparisonPolicy):
    """Drop-in for FcfsPolicy (baselines.py:108-155)."""

    name = "fcfs"


class GpuProgramPriorityPolicy(_GpuComparisonPolicy):
    """Drop-in for ProgramPriorityPolicy (baselines.py:158-208): the window
    key reads Call.served_tokens from the `served` column, refreshed for the
    ready rows every tick."""

    name = "program_priority"

    def _extra_cols(self, calls: Sequence, n: int) -> dict:
        return {"served": np.fromiter((c.served_tokens for c in calls), np.int64, n)}


class GpuTtlPolicy(_GpuComparisonPolicy):
    """Drop-in for TtlPolicy (baselines.py:211-315): unconditional pins with
    a static or EMA-scaled deadline; expired pins and the pin-first reclaim
    order run through the same device tables as MARS's."""

    def __init__(self, kind: str, pressure=None, ttl_seconds: float = 30.0,
                 multiplier: float = 1.5, window_size: int = 128, max_decode_slots: int = 64,
                 **kw) -> None:
        if kind not in ("static_ttl", "dynamic_ttl"):
            raise ValueError(f"not a ttl policy kind: {kind}")
        self.name = kind
        super().__init__(window_size, max_decode_slots, pressure=pressure,
                         ttl_seconds=float(ttl_seconds), ttl_multiplier=float(multiplier), **kw)
        self.ttl_seconds, self.multiplier = ttl_seconds, multiplier

    def retention_decision(self, call, pool, telemetry, gpu, now):
        # TtlPolicy.retention_decision (baselines.py:238-243): always pin
        if self.name == "static_ttl":
            deadline = now + self.ttl_seconds
        else:
            ema = telemetry.ema_tool_duration
            deadline = now + self.multiplier * (self._tool_prior if ema is None else ema)
        return RetentionDecision(True, 0.0, 0.0, deadline)


def make_gpu_policy(kind: str, mlfq=None, retention=None, pressure=None, params=None,
                    enable_coordinator: bool = True, enable_coscheduler: bool = True,
                    **kw):
    """make_policy (baselines.py:458-495) over the B200 drop-ins."""
    params = dict(params or {})
    window = params.pop("window_size", getattr(mlfq, "window_size", 128))
    slots = params.pop("max_decode_slots", getattr(mlfq, "max_decode_slots", 64))
    if kind == "fcfs":
        return GpuFcfsPolicy(window_size=window, max_decode_slots=slots, **kw)
    if kind == "program_priority":
        return GpuProgramPriorityPolicy(window_size=window, max_decode_slots=slots, **kw)
    if kind in ("static_ttl", "dynamic_ttl"):
        return GpuTtlPolicy(kind, pressure, ttl_seconds=params.pop("ttl_seconds", 30.0),
                            multiplier=params.pop("multiplier", 1.5), window_size=window,
                            max_decode_slots=slots, **kw)
    if kind == "mars":
        return GpuMarsPolicy(mlfq, retention, pressure, enable_coordinator=enable_coordinator,
                             enable_coscheduler=enable_coscheduler, **kw)
    raise ValueError(f"unknown policy kind {kind!r}")
