"""Host-side handle on one device replica of the MARS session table.

``MarsEngine`` owns a ``mars_ctx`` (include/mars_b200.h): the structure-of-
arrays session table in HBM, the admission list, the pool/telemetry/controller
scalars, and the step pipeline.  It is the device-resident engine mode the
benchmark and the multi-GPU replicas use; the reference-plugin drop-in
(``policy.GpuMarsPolicy``) drives the same context one tick at a time.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import _native as N
from .snapshot import COLUMNS, F_LONG, Snapshot

JOURNAL_NAMES = {1: "alloc", 2: "free", 3: "free", 4: "free"}


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


_COL_INDEX = {name: i for i, name in enumerate(N.COL_FIELDS)}  # mars_cols field order
assert [f for f, _ in N.MarsCols._fields_] == list(N.COL_FIELDS.values())
_P_COLS = C.POINTER(N.MarsCols)

_CT = {np.uint8: C.c_uint8, np.uint32: C.c_uint32, np.int32: C.c_int32, np.int64: C.c_int64,
       np.float64: C.c_double}


def step_columns(policy: str = "mars", enable_coordinator: bool = True, mode: int = 0):
    """The session-table columns a step reads in this configuration -- what a
    caller holding the state on the host must upload before each step
    (mars_upsert_rows).  ``arrival`` is the order key only with the coordinator
    off (scheduler.py:391-392 ablation) or for the comparison policies, and
    admission stamps ``now`` instead (baselines.py:351-356); ``served`` is read
    by charge_service (SERVICE / ADVANCE) and program_priority's key;
    ``rounds_left`` only by the tick's tail (ADVANCE)."""
    skip = set()
    if policy == "mars" and enable_coordinator:
        skip.add("arrival")
    if policy != "program_priority" and not (mode & (N.MODE_SERVICE | N.MODE_ADVANCE)):
        skip.add("served")
    if not (mode & N.MODE_ADVANCE):
        skip.add("rounds_left")
    return [k for k in COLUMNS if k not in skip]


def make_config(enable_coordinator: bool = True, enable_coscheduler: bool = True,
                initial_window: Optional[float] = None, policy: str = "mars",
                **overrides) -> N.MarsConfig:
    lib = N.load()
    cfg = N.MarsConfig()
    lib.mars_config_default(C.byref(cfg))
    cfg.policy = N.POLICY_CODES[policy]
    cfg.enable_coordinator = int(bool(enable_coordinator))
    cfg.enable_coscheduler = int(bool(enable_coscheduler))
    if initial_window is not None:
        cfg.initial_window = float(initial_window)
    for k, v in overrides.items():
        setattr(cfg, k, v)
    return cfg


@dataclass
class StepResult:
    status: int
    expired_rows: np.ndarray
    expired_blocks: np.ndarray
    admitted_rows: np.ndarray
    window_rows: np.ndarray
    decode_rows: np.ndarray
    prefill_rows: np.ndarray
    prefill_grants: np.ndarray
    evict_rows: np.ndarray
    evict_kind: np.ndarray
    evict_blocks: np.ndarray
    journal_op: np.ndarray
    journal_row: np.ndarray
    journal_n: np.ndarray
    ret_rows: np.ndarray
    ret_pin: np.ndarray
    ret_benefit: np.ndarray
    ret_cost: np.ndarray
    ret_deadline: np.ndarray
    decode_level: np.ndarray
    prefill_level: np.ndarray
    fin_rows: np.ndarray
    fin_pin: np.ndarray
    fin_benefit: np.ndarray
    fin_cost: np.ndarray
    fin_deadline: np.ndarray
    end_rows: np.ndarray   # MARS_MODE_ADVANCE: rounds that ended (decode order)
    end_kind: np.ndarray   # 0 done, 1 pinned -> tool, 2 freed -> tool
    end_blocks: np.ndarray     # blocks pinned or freed at the round's end
    end_pin: np.ndarray        # the retention decision (when the policy makes one)
    end_benefit: np.ndarray
    end_cost: np.ndarray
    end_deadline: np.ndarray
    prefill_done: np.ndarray   # MARS_MODE_ADVANCE: the grant finished the prefill
    plan_pre_charge: np.ndarray  # MARS_MODE_SERVICE: (served << 8) | level before the charge
    n_ready: int
    n_promoted: int
    pack_mode: int
    total_tokens: int
    free_after_expiry: int
    free_blocks: int
    limit: int
    slots: int
    diag: Dict[str, int] = field(default_factory=dict)


# (array, count field, dtype) of every mars_step_out array, with the byte
# offsets of its pointer (in 8-byte units) and count (4-byte units)
_OUT_ARRAYS = [
    ("expired_rows", "n_expired", np.uint32), ("expired_blocks", "n_expired", np.int32),
    ("admitted_rows", "n_admitted", np.uint32), ("window_rows", "n_window", np.uint32),
    ("decode_rows", "n_decode", np.uint32), ("prefill_rows", "n_prefill", np.uint32),
    ("prefill_grants", "n_prefill", np.int32), ("evict_rows", "n_evict", np.uint32),
    ("evict_kind", "n_evict", np.uint8), ("evict_blocks", "n_evict", np.int32),
    ("journal_op", "n_journal", np.uint8), ("journal_row", "n_journal", np.uint32),
    ("journal_n", "n_journal", np.int32), ("ret_rows", "n_retention", np.uint32),
    ("ret_pin", "n_retention", np.uint8), ("ret_benefit", "n_retention", np.float64),
    ("ret_cost", "n_retention", np.float64), ("ret_deadline", "n_retention", np.float64),
    ("decode_level", "n_decode", np.uint8), ("prefill_level", "n_prefill", np.uint8),
    ("fin_rows", "n_finish", np.uint32), ("fin_pin", "n_finish", np.uint8),
    ("fin_benefit", "n_finish", np.float64), ("fin_cost", "n_finish", np.float64),
    ("fin_deadline", "n_finish", np.float64), ("end_rows", "n_round_end", np.uint32),
    ("end_kind", "n_round_end", np.uint8), ("end_blocks", "n_round_end", np.int32),
    ("end_pin", "n_round_end", np.uint8), ("end_benefit", "n_round_end", np.float64),
    ("end_cost", "n_round_end", np.float64), ("end_deadline", "n_round_end", np.float64),
    ("prefill_done", "n_prefill", np.uint8),
]
_OUT_SPEC = [(a, getattr(N.MarsStepOut, a).offset // 8, getattr(N.MarsStepOut, c).offset // 4,
              np.dtype(d), np.dtype(d).itemsize) for a, c, d in _OUT_ARRAYS]


def _arr(p, n, dt):
    if n <= 0:
        return np.zeros(0, dtype=dt)
    return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True)


class MarsEngine:
    """One device replica (one ``mars_ctx``)."""

    def __init__(self, max_rows: int, max_queue: Optional[int] = None, device: int = 0,
                 config: Optional[N.MarsConfig] = None) -> None:
        self.lib = N.load()
        self.cfg = config if config is not None else make_config()
        self.max_rows = int(max_rows)
        self.max_queue = int(max_queue if max_queue is not None else max_rows)
        ctx = C.c_void_p()
        N.check(self.lib.mars_create(C.byref(self.cfg), device, self.max_rows, self.max_queue,
                                     C.byref(ctx)))
        self.ctx = ctx
        self.n_rows = 0
        self._out = None

    def close(self) -> None:
        if self.ctx:
            self.lib.mars_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int) -> None:
        N.check(rc, self.ctx)

    # -- session-state store -------------------------------------------------

    def upsert(self, cols: Dict[str, np.ndarray], rows: Optional[np.ndarray] = None) -> None:
        # the mars_cols struct as a raw array of 20 pointers (the drop-in calls
        # this every tick: no ctypes pointer objects per column)
        ptrs = np.zeros(len(_COL_INDEX), np.uint64)
        keep = []
        n = None
        for name, v in cols.items():
            ci = _COL_INDEX.get(name)
            if ci is None:
                continue
            a = np.ascontiguousarray(v, dtype=COLUMNS[name])
            keep.append(a)
            ptrs[ci] = a.ctypes.data
            if n is None:
                n = len(a)
            elif len(a) != n:
                raise ValueError("column lengths differ")
        if n is None:
            return
        mc = ptrs.ctypes.data_as(_P_COLS)
        if rows is None:
            self._check(self.lib.mars_upsert_rows(self.ctx, n, None, mc))
            self.n_rows = max(self.n_rows, n)
        else:
            r = np.ascontiguousarray(rows, dtype=np.int64)
            if len(r) != n:
                raise ValueError("rows / column length mismatch")
            self._check(self.lib.mars_upsert_rows(self.ctx, n, r.ctypes.data, mc))
            if n:
                self.n_rows = max(self.n_rows, int(r.max()) + 1)

    def input_arena(self) -> Dict[str, np.ndarray]:
        """The library's pinned input arena (mars_input_arena): one writable
        numpy view per column (``max_rows`` rows), laid out like the device
        table, for callers that keep the whole table on the host and upload
        it every step (``upsert_arena``)."""
        if getattr(self, "_in_views", None) is None:
            base, size = C.c_void_p(), C.c_int64()
            mc = N.MarsCols()
            self._check(self.lib.mars_input_arena(self.ctx, C.byref(base), C.byref(size),
                                                  C.byref(mc)))
            views = {}
            for name, field in N.COL_FIELDS.items():
                dt = np.dtype(COLUMNS[name])
                addr = C.cast(getattr(mc, field), C.c_void_p).value
                buf = (C.c_uint8 * (self.max_rows * dt.itemsize)).from_address(addr)
                views[name] = np.frombuffer(buf, dtype=dt)
            self._in_views = views
        return self._in_views

    def upsert_arena(self, n: int, names) -> None:
        """Rows [0, n) of the named columns from the input arena to the table
        (mars_upsert_arena: one pitched copy per run of adjacent columns)."""
        mask = 0
        for i, name in enumerate(N.COL_FIELDS):
            if name in names:
                mask |= 1 << i
        self._check(self.lib.mars_upsert_arena(self.ctx, int(n), mask))
        self.n_rows = max(self.n_rows, int(n))

    def read(self, names=None, rows: Optional[np.ndarray] = None) -> Dict[str, np.ndarray]:
        names = list(names or N.COL_FIELDS)
        n = self.n_rows if rows is None else len(rows)
        out = {k: np.zeros(n, dtype=COLUMNS[k]) for k in names}
        mc = N.MarsCols()
        for k in names:
            setattr(mc, N.COL_FIELDS[k], _ptr(out[k], _CT[COLUMNS[k]]))
        if rows is None:
            self._check(self.lib.mars_read_rows(self.ctx, n, None, C.byref(mc)))
        else:
            r = np.ascontiguousarray(rows, dtype=np.int64)
            self._check(self.lib.mars_read_rows(self.ctx, n, r.ctypes.data_as(C.c_void_p),
                                                C.byref(mc)))
        return out

    def set_queue(self, rows: np.ndarray, req: np.ndarray, is_long: np.ndarray) -> None:
        r = np.ascontiguousarray(rows, dtype=np.uint32)
        q = np.ascontiguousarray(req, dtype=np.int32)
        lg = np.ascontiguousarray(is_long, dtype=np.uint8)
        self._check(self.lib.mars_set_queue(self.ctx, len(r), r.ctypes.data_as(C.c_void_p),
                                            q.ctypes.data_as(C.c_void_p),
                                            lg.ctypes.data_as(C.c_void_p)))

    def queue_append(self, rows: np.ndarray, req: np.ndarray, is_long: np.ndarray) -> None:
        """Arrivals to the end of the device admission list."""
        r = np.ascontiguousarray(rows, np.uint32)
        q = np.ascontiguousarray(req, np.int32)
        lg = np.ascontiguousarray(is_long, np.uint8)
        self._check(self.lib.mars_queue_append(self.ctx, len(r), r.ctypes.data_as(C.c_void_p),
                                               q.ctypes.data_as(C.c_void_p),
                                               lg.ctypes.data_as(C.c_void_p)))

    def on_admit(self, rows, r0_prefill, now) -> None:
        """MarsPolicy.on_admit for a batch of rows, on the device (mars_on_admit)."""
        r = np.ascontiguousarray(rows, np.int64)
        p = np.ascontiguousarray(r0_prefill, np.int32)
        t = np.ascontiguousarray(np.broadcast_to(np.asarray(now, np.float64), r.shape))
        self._check(self.lib.mars_on_admit(self.ctx, len(r), r.ctypes.data_as(C.c_void_p),
                                           p.ctypes.data_as(C.c_void_p),
                                           t.ctypes.data_as(C.c_void_p)))

    def get_queue(self) -> np.ndarray:
        n = C.c_int64()
        self._check(self.lib.mars_get_queue(self.ctx, 0, None, C.byref(n)))
        out = np.zeros(n.value, dtype=np.uint32)
        if n.value:
            self._check(self.lib.mars_get_queue(self.ctx, n.value, out.ctypes.data_as(C.c_void_p),
                                                C.byref(n)))
        return out

    def set_scalars(self, s: N.MarsScalars) -> None:
        self._check(self.lib.mars_set_scalars(self.ctx, C.byref(s)))

    def get_scalars(self) -> N.MarsScalars:
        s = N.MarsScalars()
        self._check(self.lib.mars_get_scalars(self.ctx, C.byref(s)))
        return s

    def load_snapshot(self, snap: Snapshot) -> None:
        if snap.n > self.max_rows:
            raise ValueError("snapshot larger than the engine's row capacity")
        self._check(self.lib.mars_set_rows(self.ctx, snap.n))
        self.upsert(snap.cols)
        self.n_rows = snap.n
        q = snap.queue
        self.set_queue(q, snap.cols["req_blocks"][q],
                       (snap.cols["flags"][q] & F_LONG) != 0)
        s = N.MarsScalars()
        s.total_blocks = snap.total_blocks
        s.free_blocks = snap.free_blocks
        s.available_kv = snap.free_blocks
        s.w_adm = float(snap.initial_window)
        s.last_update = 0.0
        s.has_ema_tool = int(snap.ema_tool is not None)
        s.ema_tool = float(snap.ema_tool or 0.0)
        s.has_ema_blocks = int(snap.ema_blocks is not None)
        s.ema_blocks = float(snap.ema_blocks or 0.0)
        s.has_blocks_seed = int(snap.blocks_seed is not None)
        s.blocks_seed = float(snap.blocks_seed or 0.0)
        s.queue_len = len(q)
        for k, v in snap.telemetry.items():
            setattr(s, k, int(v))
        self.set_scalars(s)
        # rows laid out in session-id order: expired pins come out of the scan
        # already in expired_pins() order (no sort pass)
        self.rank_ordered = bool(np.array_equal(snap.cols["rank"],
                                                np.arange(snap.n, dtype=np.uint32)))

    # -- the step ----------------------------------------------------------------

    rank_ordered = False

    def step_in(self, now: float, control_due: bool = True, active_tools: int = 0,
                queued_tools: int = 0, worker_slots: int = 8, mode: int = 0) -> N.MarsStepIn:
        si = N.MarsStepIn()
        si.now = float(now)
        si.control_due = int(bool(control_due))
        si.active_tools = int(active_tools)
        si.queued_tools = int(queued_tools)
        si.worker_slots = int(worker_slots)
        si.mode = int(mode) | (N.MODE_RANK_ORDERED if self.rank_ordered else 0)
        return si

    def set_config(self, cfg: N.MarsConfig) -> None:
        """Replaces the configuration (same policy) of a live context."""
        self._check(self.lib.mars_set_config(self.ctx, C.byref(cfg)))
        self.cfg = cfg

    def set_graph(self, on: bool) -> None:
        self._check(self.lib.mars_set_graph(self.ctx, int(bool(on))))

    def enqueue(self, si: N.MarsStepIn) -> None:
        self._check(self.lib.mars_step_enqueue(self.ctx, C.byref(si)))

    def fetch(self, copy: bool = True) -> StepResult:
        """The step's outputs.  ``copy=False``: the arrays are views of the
        pinned output arena the device wrote (no host memcpy), valid until
        the next fetch overwrites it."""
        if self._out is None:
            self._fetch_setup()
        o = self._out
        self._check(self.lib.mars_step_fetch(self.ctx, C.byref(o)))
        i32, p64, arena, base = self._out_i32, self._out_p64, self._arena, self._arena_base
        arrs = {}
        for name, po, co, dt, isz in _OUT_SPEC:
            n = int(i32[co])
            p = int(p64[po]) if n > 0 else 0
            if p == 0:
                arrs[name] = np.empty(0, dt)
            else:
                s0 = p - base
                v = arena[s0:s0 + n * isz].view(dt)
                arrs[name] = v.copy() if copy else v
        npc = int(o.n_decode) + int(o.n_prefill)
        if o.plan_pre_charge and npc:
            s0 = int(C.cast(o.plan_pre_charge, C.c_void_p).value) - base
            v = arena[s0:s0 + npc * 8].view(np.int64)
            arrs["plan_pre_charge"] = v.copy() if copy else v
        else:
            arrs["plan_pre_charge"] = np.empty(0, np.int64)
        return StepResult(
            status=o.status, **arrs,
            n_ready=o.n_ready, n_promoted=o.n_promoted, pack_mode=o.pack_mode,
            total_tokens=o.total_tokens, free_after_expiry=o.free_after_expiry,
            free_blocks=o.free_blocks, limit=o.limit, slots=o.slots,
            diag={"n_window_cand": o.n_window_cand, "n_victim_cand": o.n_victim_cand,
                  "walk_slow": o.walk_slow, "sort_path": o.sort_path,
                  "n_round_end": o.n_round_end, "n_done": o.n_done,
                  "n_fullscan": o.n_fullscan, "ref_flags": o.ref_flags,
                  "ref_rounds": o.ref_rounds, "n_window_ref": o.n_window_ref,
                  "n_victim_ref": o.n_victim_ref})

    def _fetch_setup(self) -> None:
        base, size = C.c_void_p(), C.c_int64()
        self._check(self.lib.mars_output_arena(self.ctx, C.byref(base), C.byref(size)))
        self._arena_base = int(base.value)
        self._arena = np.ctypeslib.as_array((C.c_uint8 * int(size.value)).from_address(
            self._arena_base))
        self._out = N.MarsStepOut()
        raw = np.frombuffer(self._out, np.uint8)
        self._out_i32 = raw[:len(raw) // 4 * 4].view(np.int32)
        self._out_p64 = raw[:len(raw) // 8 * 8].view(np.uint64)

    def fetch_reference(self) -> StepResult:
        """The field-by-field conversion (kept for the tests that check the
        fast path against it)."""
        o = N.MarsStepOut()
        self._check(self.lib.mars_step_fetch(self.ctx, C.byref(o)))
        return StepResult(
            status=o.status,
            expired_rows=_arr(o.expired_rows, o.n_expired, np.uint32),
            expired_blocks=_arr(o.expired_blocks, o.n_expired, np.int32),
            admitted_rows=_arr(o.admitted_rows, o.n_admitted, np.uint32),
            window_rows=_arr(o.window_rows, o.n_window, np.uint32),
            decode_rows=_arr(o.decode_rows, o.n_decode, np.uint32),
            prefill_rows=_arr(o.prefill_rows, o.n_prefill, np.uint32),
            prefill_grants=_arr(o.prefill_grants, o.n_prefill, np.int32),
            evict_rows=_arr(o.evict_rows, o.n_evict, np.uint32),
            evict_kind=_arr(o.evict_kind, o.n_evict, np.uint8),
            evict_blocks=_arr(o.evict_blocks, o.n_evict, np.int32),
            journal_op=_arr(o.journal_op, o.n_journal, np.uint8),
            journal_row=_arr(o.journal_row, o.n_journal, np.uint32),
            journal_n=_arr(o.journal_n, o.n_journal, np.int32),
            ret_rows=_arr(o.ret_rows, o.n_retention, np.uint32),
            ret_pin=_arr(o.ret_pin, o.n_retention, np.uint8),
            ret_benefit=_arr(o.ret_benefit, o.n_retention, np.float64),
            ret_cost=_arr(o.ret_cost, o.n_retention, np.float64),
            ret_deadline=_arr(o.ret_deadline, o.n_retention, np.float64),
            decode_level=_arr(o.decode_level, o.n_decode, np.uint8),
            prefill_level=_arr(o.prefill_level, o.n_prefill, np.uint8),
            fin_rows=_arr(o.fin_rows, o.n_finish, np.uint32),
            fin_pin=_arr(o.fin_pin, o.n_finish, np.uint8),
            fin_benefit=_arr(o.fin_benefit, o.n_finish, np.float64),
            fin_cost=_arr(o.fin_cost, o.n_finish, np.float64),
            fin_deadline=_arr(o.fin_deadline, o.n_finish, np.float64),
            end_rows=_arr(o.end_rows, o.n_round_end, np.uint32),
            end_kind=_arr(o.end_kind, o.n_round_end, np.uint8),
            end_blocks=_arr(o.end_blocks, o.n_round_end, np.int32),
            end_pin=_arr(o.end_pin, o.n_round_end, np.uint8),
            end_benefit=_arr(o.end_benefit, o.n_round_end, np.float64),
            end_cost=_arr(o.end_cost, o.n_round_end, np.float64),
            end_deadline=_arr(o.end_deadline, o.n_round_end, np.float64),
            prefill_done=_arr(o.prefill_done, o.n_prefill if o.prefill_done else 0, np.uint8),
            plan_pre_charge=_arr(o.plan_pre_charge,
                                 (o.n_decode + o.n_prefill) if o.plan_pre_charge else 0, np.int64),
            n_ready=o.n_ready, n_promoted=o.n_promoted, pack_mode=o.pack_mode,
            total_tokens=o.total_tokens, free_after_expiry=o.free_after_expiry,
            free_blocks=o.free_blocks, limit=o.limit, slots=o.slots,
            diag={"n_window_cand": o.n_window_cand, "n_victim_cand": o.n_victim_cand,
                  "walk_slow": o.walk_slow, "sort_path": o.sort_path,
                  "n_round_end": o.n_round_end, "n_done": o.n_done,
                  "n_fullscan": o.n_fullscan, "ref_flags": o.ref_flags,
                  "ref_rounds": o.ref_rounds, "n_window_ref": o.n_window_ref,
                  "n_victim_ref": o.n_victim_ref})

    def step(self, si: N.MarsStepIn) -> StepResult:
        self.enqueue(si)
        return self.fetch()

    def retention_batch(self, context: np.ndarray, kv: np.ndarray, total_blocks: int,
                        usage: float, ema: float, now: float):
        ctx = np.ascontiguousarray(context, dtype=np.int32)
        kvv = np.ascontiguousarray(kv, dtype=np.int32)
        n = len(ctx)
        pin = np.zeros(n, np.uint8)
        b, c, d = (np.zeros(n, np.float64) for _ in range(3))
        self._check(self.lib.mars_retention_batch(
            self.ctx, n, ctx.ctypes.data_as(C.c_void_p), kvv.ctypes.data_as(C.c_void_p),
            int(total_blocks), float(usage), float(ema), float(now),
            pin.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
            c.ctypes.data_as(C.c_void_p), d.ctypes.data_as(C.c_void_p)))
        return pin.astype(bool), b, c, d

    def checkpoint(self) -> None:
        self._check(self.lib.mars_checkpoint(self.ctx))

    def restore(self) -> None:
        self._check(self.lib.mars_restore(self.ctx))

    def flush_l2(self, nbytes: int) -> None:
        self._check(self.lib.mars_flush_l2(self.ctx, int(nbytes)))

    def set_profiling(self, on: bool) -> None:
        self._check(self.lib.mars_set_profiling(self.ctx, int(bool(on))))

    def resume(self, rows, finish_time, duration, new_prefill, decode_tokens,
               now: float) -> Dict[str, int]:
        """resume_from_tool (sim.py:190-231) for tools that finished, in the tool
        plane's finish order (mars_resume)."""
        rows = np.ascontiguousarray(rows, np.int64)
        fin = np.ascontiguousarray(finish_time, np.float64)
        dur = np.ascontiguousarray(duration, np.float64)
        newp = np.ascontiguousarray(new_prefill, np.int32)
        dec = np.ascontiguousarray(decode_tokens, np.int32)
        cnt = np.zeros(3, np.int32)
        self._check(self.lib.mars_resume(self.ctx, len(rows), rows.ctypes.data, fin.ctypes.data,
                                         dur.ctypes.data, newp.ctypes.data, dec.ctypes.data,
                                         float(now), cnt.ctypes.data))
        return {"warm": int(cnt[0]), "cold": int(cnt[1]), "evicted": int(cnt[2])}

    def resume_rows(self, n: int) -> Dict[str, np.ndarray]:
        """Per row of the last ``resume`` (mars_resume_rows): ``kind`` 0 warm,
        1 cold, 2 cold after the return-time release of an expired pin;
        ``blocks`` unpinned or released; the gpu_submit payload's ``context``,
        ``need`` (required_prefill) and ``projected`` blocks (sim.py:190-231)."""
        out = {k: np.zeros(n, np.int32) for k in ("blocks", "context", "need", "projected")}
        out["kind"] = np.zeros(n, np.uint8)
        self._check(self.lib.mars_resume_rows(
            self.ctx, n, out["kind"].ctypes.data, out["blocks"].ctypes.data,
            out["context"].ctypes.data, out["need"].ctypes.data, out["projected"].ctypes.data))
        return out

    def kernel_times(self) -> Dict[str, float]:
        ms = (C.c_float * len(N.KTIME_NAMES))()
        self._check(self.lib.mars_kernel_times(self.ctx, ms, len(N.KTIME_NAMES)))
        return {k: float(v) for k, v in zip(N.KTIME_NAMES, ms)}

    def launches(self) -> int:
        return int(self.lib.mars_last_launch_count(self.ctx))


def canonical(res: StepResult, eng: MarsEngine, snap: Snapshot, control_due: bool = True) -> dict:
    """Device step result in the oracle's canonical layout (oracle/snapshot_step.py)."""
    sc = eng.get_scalars()
    kinds = {0: "running", 1: "pinned"}
    exp = [(int(r), int(b)) for r, b in zip(res.expired_rows, res.expired_blocks)]
    out = dict(
        expired=exp,
        expiry_journal=[("free", r, b, True) for r, b in exp],
        probe=dict(available_kv=int(res.free_after_expiry), usage=float(sc.kv_usage_ratio),
                   active_sessions=int(sc.active_sessions)),
        control=None,
        retention=[],
        window=[int(x) for x in res.window_rows],
        decodes=[int(x) for x in res.decode_rows],
        prefills=[(int(r), int(g)) for r, g in zip(res.prefill_rows, res.prefill_grants)],
        evictions=[(int(r), kinds[int(k)], int(b))
                   for r, k, b in zip(res.evict_rows, res.evict_kind, res.evict_blocks)],
        total_tokens=int(res.total_tokens),
        journal=[(JOURNAL_NAMES[int(o)], int(r), int(n), int(o) == 3)
                 for o, r, n in zip(res.journal_op, res.journal_row, res.journal_n)],
        free_blocks=int(res.free_blocks),
        n_ready=int(res.n_ready) + len(res.admitted_rows),
    )
    if control_due:
        out["control"] = dict(
            w_adm=float(sc.w_adm), last_update=float(sc.last_update), limit=int(res.limit),
            slots=int(res.slots), admitted=[int(x) for x in res.admitted_rows],
            queue=[int(x) for x in eng.get_queue()],
            cpu_overloaded=bool(sc.cpu_overloaded), kv_overloaded=bool(sc.kv_overloaded),
            streaks=(int(sc.cpu_high_streak), int(sc.cpu_low_streak), int(sc.kv_high_streak),
                     int(sc.kv_low_streak)),
            blocks_seed=(float(sc.blocks_seed) if sc.has_blocks_seed else None),
            available_kv=int(sc.available_kv))
    order = np.argsort(res.ret_rows, kind="stable")
    out["retention"] = [(int(res.ret_rows[i]), bool(res.ret_pin[i]), float(res.ret_benefit[i]),
                         float(res.ret_cost[i]), float(res.ret_deadline[i])) for i in order]
    st = eng.read(["phase", "flags", "level", "promos", "wait_since", "ready_since", "context",
                   "kv", "rem_decode", "preempt", "served"])
    out["state"] = st
    return out
