"""A whole trace with the tick on the B200.

``run_device_simulation`` replays the reference tick loop
(agentsched/sim.py:90-431, ``run_simulation``) with every per-session
transition on the device: the scheduling half (``mars_step``: pin expiry,
probe, refresh_pressure + balance_and_admit + admit, MLFQ aging, window,
build_plan with reclamation), the tick's tail (``MARS_MODE_ADVANCE``:
step_gpu, charge_service, each ending round's retention / pin / free / DONE)
and resume_from_tool (``mars_resume``).  The host keeps what is trace data or
a scalar: arrivals (row upserts + the admission-list append), the tool plane
(``ToolPlane``, engine.py:366-442: worker slots and the FIFO overflow, whose
counts feed the probe), the control cadence, and the idle-tick jump.

It returns the reference's run counters (sim.py:137-146) and the final clock,
which the tests compare with the frozen reference runs.  Given an
``EventLog`` it also writes the reference's JSONL event log (engine.py:77-104,
SURVEY §8(f) row 2): every record the reference's tick loop emits, in its
order, serialised on the host from the device's per-step outputs -- the
expiry list, the admission prefix, the plan's ordered alloc / evict journal,
the plan, prefill completions, each ended round's blocks and retention
decision, and each resume's warm / cold outcome -- so the log of a device
run is byte-identical to the reference's.
"""

from __future__ import annotations

import heapq
import json
import math
from dataclasses import dataclass
from typing import Dict, List, NamedTuple, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .engine import MarsEngine, make_config
from .snapshot import COLUMNS, F_LONG, F_QUEUED

WAITING_ADMISSION, EMPTY = 0, 7


@dataclass
class FinishedTool:
    row: int
    start_time: float
    finish_time: float
    duration_s: float
    enqueue_time: float


class EventLog:
    """The reference's append-only event log (engine.py:77-104): records
    ``{"t", "seq", "kind", "session_id", **payload}`` with ``seq`` from 1,
    serialised as compact JSON lines in insertion order."""

    def __init__(self) -> None:
        self.records: List[dict] = []

    def emit(self, t: float, kind: str, sid: Optional[str] = None, **payload) -> None:
        rec = {"t": t, "seq": len(self.records) + 1, "kind": kind, "session_id": sid}
        rec.update(payload)
        self.records.append(rec)

    def jsonl_bytes(self) -> bytes:
        return b"".join((json.dumps(r, separators=(",", ":")) + "\n").encode()
                        for r in self.records)


class _Telemetry:
    """The host's view of the reference Telemetry fields that the log shows
    (telemetry.py:96-120 record, :152-158 probe): what the tick's probe set,
    plus the drift of the events recorded after it."""

    def __init__(self, total: int) -> None:
        self.available_kv = total
        self.kv_usage_ratio = 0.0
        self.active_tools = self.queued_tools = self.active_sessions = 0

    def probe(self, free: int, total: int, tools: "ToolPlane", active: int) -> None:
        self.available_kv = free
        self.kv_usage_ratio = (total - free) / total
        self.active_tools = tools.active_count()
        self.queued_tools = tools.queued_count()
        self.active_sessions = active

    def snapshot(self, sc) -> dict:
        return {
            "available_kv": self.available_kv,
            "kv_usage_ratio": self.kv_usage_ratio,
            "active_tools": self.active_tools,
            "queued_tools": self.queued_tools,
            "ema_tool_duration_s": float(sc.ema_tool) if sc.has_ema_tool else None,
            "ema_blocks_per_session": float(sc.ema_blocks) if sc.has_ema_blocks else None,
            "active_sessions": self.active_sessions,
            "cpu_overloaded": bool(sc.cpu_overloaded),
            "kv_overloaded": bool(sc.kv_overloaded),
        }


class ToolPlane:
    """engine.py:366-442: fixed worker slots plus a FIFO overflow queue; a
    freed slot goes to the oldest queued tool, started at the instant the
    slot freed (or its enqueue instant, if later)."""

    def __init__(self, worker_slots: int) -> None:
        if worker_slots < 1:
            raise ValueError("tool plane needs at least one worker slot")
        self.worker_slots = worker_slots
        self._running: List[Tuple[float, int, int, float, float, float]] = []
        self._queued: List[Tuple[int, float, float]] = []
        self._seq = 0
        self.promoted: List[Tuple[int, float, float]] = []   # (row, start, duration)

    def active_count(self) -> int:
        return len(self._running)

    def queued_count(self) -> int:
        return len(self._queued)

    def next_finish_time(self) -> Optional[float]:
        return self._running[0][0] if self._running else None

    def start_tool(self, row: int, duration_s: float, now: float) -> bool:
        if duration_s < 0:
            raise N.ContractViolation("tool duration must be >= 0")
        if len(self._running) < self.worker_slots:
            self._seq += 1
            heapq.heappush(self._running, (now + duration_s, self._seq, row, now, duration_s, now))
            return True
        self._queued.append((row, duration_s, now))
        return False

    def complete_tools(self, now: float) -> List[FinishedTool]:
        done: List[FinishedTool] = []
        while self._running and self._running[0][0] <= now:
            finish, _, row, start, dur, enq = heapq.heappop(self._running)
            done.append(FinishedTool(row, start, finish, dur, enq))
            if self._queued:
                qrow, qdur, qenq = self._queued.pop(0)
                qstart = max(finish, qenq)
                self._seq += 1
                heapq.heappush(self._running, (qstart + qdur, self._seq, qrow, qstart, qdur, qenq))
                self.promoted.append((qrow, qstart, qdur))
        return done

    def take_promotions(self) -> List[Tuple[int, float, float]]:
        out, self.promoted = self.promoted, []
        return out


def run_device_simulation(traces: Sequence, total_blocks: int, tool_worker_slots: int,
                          policy: str = "mars", enable_coordinator: bool = True,
                          enable_coscheduler: bool = True, enable_control_plane: bool = True,
                          initial_window: Optional[float] = None, device: int = 0,
                          max_ticks: int = 5_000_000,
                          log: Optional[EventLog] = None,
                          kv_state: Optional[dict] = None,
                          kv_tier: Optional[dict] = None) -> Tuple[Dict[str, int], float]:
    """``policy`` (a POLICY_KINDS name) over ``traces`` (objects with
    session_id, arrival_time_s and rounds of new_prefill_tokens /
    decode_tokens / tool_duration_s, as agentsched.workload.Trace).  MARS
    admits through its control plane unless ``enable_control_plane`` is off;
    the comparison policies admit at arrival (sim.py:116).  Returns
    (counters, final clock); fills ``log`` with the run's event log when
    one is given.  With ``kv_state`` (a dict) the device block-ID manager
    rides along (every alloc / free of the run applied to concrete block IDs
    on the device, mars_kv) and its final free-stack order is stored there
    as ``kv_state["top"]`` (with ``depth``, ``fresh``, ``status``).

    ``kv_tier`` (a dict, with ``kv_state``): the KV bytes follow the run's
    decisions through a pinned host ring (``block_bytes``, ``host_blocks``;
    decision-neutral, the reference has no host tier): a pin
    copies the session's table to the host (sim.py:261-265), a warm resume
    copies it back (sim.py:193-200), and a running session's eviction or an
    unpinned tool boundary copies the freed blocks out (captured on the
    device as the step frees them).  Blocks, bytes and copy times per
    direction are stored back into the dict; ``verify=True`` also records
    which block every host slot holds (``slot_ids``)."""
    order = sorted(traces, key=lambda t: (t.arrival_time_s, t.session_id))
    n = len(order)
    cfg = make_config(enable_coordinator, enable_coscheduler, initial_window=initial_window,
                      policy=policy)
    cfg_admission = enable_control_plane and policy == "mars"
    bs = int(cfg.block_size)
    for tr in order:  # sim.py:103-109
        ctx = sum(r.new_prefill_tokens + r.decode_tokens for r in tr.rounds)
        if -(-ctx // bs) > total_blocks:
            raise N.ContractViolation(f"session {tr.session_id} cannot fit the pool")
    eng = MarsEngine(max_rows=max(n, 1), max_queue=max(n, 1), device=device, config=cfg)
    decides = (policy == "mars" and enable_coscheduler) or policy in ("static_ttl", "dynamic_ttl")
    try:
        kv = None
        if kv_state is not None:
            from .kvstore import KvBlockManager
            most = max((-(-sum(r.new_prefill_tokens + r.decode_tokens for r in tr.rounds) // bs)
                        for tr in order), default=1)
            if kv_tier is not None:
                kv = KvBlockManager(eng, total_blocks, max_blocks_per_row=max(most, 1),
                                    block_bytes=int(kv_tier["block_bytes"]), layers=1,
                                    host_blocks=int(kv_tier.get("host_blocks", 2 * total_blocks)))
                if kv_tier.get("pattern"):
                    _fill_pattern(kv)
                kv.capture(True)
            else:
                kv = KvBlockManager(eng, total_blocks, max_blocks_per_row=max(most, 1))
        tier = _HostTier(kv, kv_tier) if kv_tier is not None else None
        out = _run(eng, cfg, order, total_blocks, tool_worker_slots, max_ticks, cfg_admission,
                   policy, log, decides, tier)
        if tier is not None:
            tier.finish()
        if kv is not None:
            top, depth, fresh, status = kv.state(total_blocks)
            kv_state.update(top=top, depth=depth, fresh=fresh, status=status)
        return out
    finally:
        eng.close()


class TraceRound(NamedTuple):
    new_prefill_tokens: int
    decode_tokens: int
    tool_duration_s: Optional[float]


class SessionTrace(NamedTuple):
    session_id: str
    arrival_time_s: float
    rounds: Tuple[TraceRound, ...]


def load_trace(path: str) -> List[SessionTrace]:
    """A JSONL session-trace file in the reference's format
    (agentsched/workload.py:276-330: session_id, arrival_time_s, rounds of
    new_prefill_tokens / decode_tokens / tool_duration_s)."""
    out = []
    with open(path, "r", encoding="utf-8") as fh:
        for line in fh:
            if not line.strip():
                continue
            rec = json.loads(line)
            out.append(SessionTrace(
                str(rec["session_id"]), float(rec["arrival_time_s"]),
                tuple(TraceRound(int(r["new_prefill_tokens"]), int(r["decode_tokens"]),
                                 None if r["tool_duration_s"] is None else float(r["tool_duration_s"]))
                      for r in rec["rounds"])))
    return out


def block_pattern(ids, block_bytes: int) -> np.ndarray:
    """Test content of pool blocks: block `id` holds its id (u32) followed
    by the byte id % 251."""
    ids = np.asarray(ids, np.uint32)
    out = np.empty((len(ids), block_bytes), np.uint8)
    out[:] = (ids % 251).astype(np.uint8)[:, None]
    out[:, :4] = ids.view(np.uint8).reshape(-1, 4)
    return out


def _fill_pattern(kv) -> None:
    """Every pool block gets block_pattern (through the host tier)."""
    host = kv.host_view()
    n = min(kv.total_blocks, kv.host_blocks)
    for a in range(0, kv.total_blocks, n):
        ids = np.arange(a, min(a + n, kv.total_blocks), dtype=np.uint32)
        host[:len(ids)] = block_pattern(ids, kv.block_bytes)
        kv.restore(ids, 0, 2)


class _HostTier:
    """The KV bytes the run's decisions imply, through the host ring."""

    def __init__(self, kv, stats: dict) -> None:
        import time
        self._time = time.perf_counter
        self.kv, self.st = kv, stats
        self.verify = bool(stats.get("verify"))
        self.slots: Dict[int, Tuple[int, int]] = {}   # pinned row -> (first slot, blocks)
        self.slot_ids: Dict[int, int] = {}            # (verify) host slot -> block id
        for k in ("evict_blocks", "pin_blocks", "restore_blocks", "d2h_s", "h2d_s"):
            stats[k] = 0
        self.bb = kv.block_bytes

    def _guard(self, s0: int, n: int) -> None:
        # a ring write over a pinned session's host copy would break its restore
        for r, (a, m) in self.slots.items():
            if s0 < a + m and a < s0 + n:
                raise RuntimeError(f"host tier too small: pinned row {r}'s copy overwritten")

    def after_step(self, res) -> None:
        # (copy times: the calls that moved blocks, each synchronous)
        t0 = self._time()
        n, s0, ids = self.kv.offload_captured(want_ids=self.verify)
        if n:
            self.st["d2h_s"] += self._time() - t0
            self._guard(s0, n)
            self.st["evict_blocks"] += n
            if self.verify:
                self.slot_ids.update(zip(range(s0, s0 + n), ids.tolist()))
        pins = [(int(r), int(b)) for r, k, b in zip(res.end_rows.tolist(), res.end_kind.tolist(),
                                                     res.end_blocks.tolist()) if k == 1 and b > 0]
        if pins:
            rows = [r for r, _ in pins]
            cnts = [b for _, b in pins]
            if self.verify:
                tabs = [self.kv.table(r) for r in rows]
            t0 = self._time()
            s0 = self.kv.offload_rows(rows, cnts)
            self.st["d2h_s"] += self._time() - t0
            self._guard(s0, sum(cnts))
            a = s0
            for i, (r, b) in enumerate(pins):
                self.slots[r] = (a, b)
                if self.verify:
                    self.slot_ids.update(zip(range(a, a + b), tabs[i].tolist()))
                a += b
            self.st["pin_blocks"] += sum(cnts)

    def after_resume(self, rows, kinds, blocks) -> None:
        warm = [(int(r), int(b)) for r, k, b in zip(rows, kinds, blocks) if k == 0 and b > 0]
        for r, k in zip(rows, kinds):
            if k != 0:
                self.slots.pop(int(r), None)   # an expired pin: its host copy is dropped
        if not warm:
            return
        t0 = self._time()
        slots = []
        for r, b in warm:
            a, m = self.slots.pop(r)
            if m != b:
                raise RuntimeError(f"warm resume of row {r}: {b} blocks, {m} offloaded")
            slots.append(a)
        self.kv.restore_rows([r for r, _ in warm], [b for _, b in warm], slots)
        self.st["restore_blocks"] += sum(b for _, b in warm)
        self.st["h2d_s"] += self._time() - t0

    def finish(self) -> None:
        st, bb = self.st, self.bb
        st["d2h_bytes"] = (st["evict_blocks"] + st["pin_blocks"]) * bb
        st["h2d_bytes"] = st["restore_blocks"] * bb
        st["d2h_gbs"] = st["d2h_bytes"] / st["d2h_s"] / 1e9 if st["d2h_s"] else None
        st["h2d_gbs"] = st["h2d_bytes"] / st["h2d_s"] / 1e9 if st["h2d_s"] else None
        if self.verify and st.get("pattern"):
            # every host slot holds the block it was given, and the pool blocks
            # (pinned tables restored in place) still hold their own content
            host = self.kv.host_view()
            slots = np.fromiter(self.slot_ids.keys(), np.int64, len(self.slot_ids))
            ids = np.fromiter(self.slot_ids.values(), np.int64, len(self.slot_ids))
            bad = 0
            for a in range(0, len(slots), 4096):
                s_, i_ = slots[a:a + 4096], ids[a:a + 4096]
                bad += int((host[s_] != block_pattern(i_, bb)).any(axis=1).sum())
            st["host_slots_checked"], st["host_slots_bad"] = len(slots), bad
            pool_bad = 0
            n = min(self.kv.total_blocks, self.kv.host_blocks)
            for a in range(0, self.kv.total_blocks, n):
                i_ = np.arange(a, min(a + n, self.kv.total_blocks), dtype=np.uint32)
                self.kv.evict(i_, 0, 2)
                pool_bad += int((host[:len(i_)] != block_pattern(i_, bb)).any(axis=1).sum())
            st["pool_blocks_bad"] = pool_bad


def _run(eng: MarsEngine, cfg, order, total_blocks: int, slots: int, max_ticks: int,
         admission: bool, policy: str, log: Optional[EventLog], decides: bool,
         tier: Optional[_HostTier] = None):
    n = len(order)
    bs = int(cfg.block_size)
    sid_rank = {sid: i for i, sid in enumerate(sorted(t.session_id for t in order))}
    r0p = np.array([t.rounds[0].new_prefill_tokens for t in order], np.int32)
    dec0 = np.array([t.rounds[0].decode_tokens for t in order], np.int32)
    req = -(-r0p.astype(np.int64) // bs)
    long_ = req > cfg.long_session_fraction * total_blocks   # control.py:91 (strict)
    eng._check(eng.lib.mars_set_rows(eng.ctx, n))
    eng.n_rows = n
    cols = {k: np.zeros(n, t) for k, t in COLUMNS.items()}
    cols.update({
        "phase": np.full(n, EMPTY, np.uint8),
        "rank": np.array([sid_rank[t.session_id] for t in order], np.uint32),
        "arrival": np.array([t.arrival_time_s for t in order], np.float64),
        "r0_prefill": r0p,
        "r0_decode": dec0,
        "req_blocks": req.astype(np.int32),
        "rounds_left": np.array([len(t.rounds) - 1 for t in order], np.int32),
    })
    eng.upsert(cols)
    eng.rank_ordered = all(sid_rank[t.session_id] == i for i, t in enumerate(order))
    s = N.MarsScalars()
    s.total_blocks = s.free_blocks = s.available_kv = total_blocks
    s.w_adm = float(cfg.initial_window)
    eng.set_scalars(s)

    sid = [t.session_id for t in order]
    tools = ToolPlane(slots)
    tel = _Telemetry(total_blocks)
    submit_t = [0.0] * n          # Call.round_submit_time (engine.py:322-330)
    first_seen = set()            # (row, round) with a first token logged (sim.py:365-371)
    tick = float(cfg.tick_duration_s)
    clock = 0.0
    next_control = 0.0
    nxt = 0
    queue: List[int] = []
    rnd = [0] * n
    active = pinned = 0
    cnt = dict(admitted=0, completed=0, evictions=0, preemptions=0, warm_resumes=0,
               cold_resumes=0, pins=0, gpu_tokens=0)

    def admit_log(r: int, now: float) -> None:  # sim.py:148-166 gpu_submit
        p = int(r0p[r])
        proj = -(-p // bs)
        log.emit(now, "gpu_submit", sid[r], round=0, arrival_time=order[r].arrival_time_s,
                 required_prefill=p, new_tokens=p, context_tokens=p, warm=None,
                 projected_blocks=proj)
        tel.available_kv -= proj
        submit_t[r] = now

    def evict_log(r: int, blocks: int, victim: str, reason: str, t: float) -> None:
        # sim.py:168-184: the pool op's observer record, then the evict record
        if victim == "pinned":
            log.emit(t, "free", sid[r], blocks=blocks, from_pinned=True)
        elif blocks > 0:
            log.emit(t, "free", sid[r], blocks=blocks)
        log.emit(t, "evict", sid[r], blocks=blocks, victim=victim, reason=reason)

    ticks = 0
    while nxt < n or queue or active:
        ticks += 1
        if ticks > max_ticks:
            raise RuntimeError(f"exceeded max_ticks={max_ticks} with work outstanding")
        now = clock
        # arrivals (sim.py:289-301): queued for admission, list order = arrival order
        new = []
        while nxt < n and order[nxt].arrival_time_s <= now + 1e-9:
            new.append(nxt)
            nxt += 1
        if new and admission:
            rows = np.array(new, np.int64)
            eng.upsert({"phase": np.full(len(new), WAITING_ADMISSION, np.uint8),
                        "flags": (F_QUEUED | np.where(long_[rows], F_LONG, 0)).astype(np.uint8)},
                       rows=rows)
            queue += new
            # appended to the device list, whose residual keeps the packed order
            eng.queue_append(rows, req[rows], long_[rows])
        elif new:
            # admit() at arrival (sim.py:148-166): submit_round + on_admit
            rows = np.array(new, np.int64)
            k = len(new)
            eng.upsert({"phase": np.full(k, 1, np.uint8), "flags": np.ones(k, np.uint8),
                        "context": r0p[rows], "rem_decode": dec0[rows],
                        "ready_since": np.full(k, now), "wait_since": np.full(k, now),
                        "level": np.zeros(k, np.uint8)}, rows=rows)
            if policy == "mars":  # on_admit: initial_level on the device
                eng.on_admit(rows, r0p[rows], now)
            cnt["admitted"] += k
            active += k
            if log is not None:
                for r in new:
                    admit_log(r, now)
        # tools that finished (sim.py:303-322): resume_from_tool on the device
        done = tools.complete_tools(now)
        if log is not None:
            for r, start, dur in tools.take_promotions():
                log.emit(start, "tool_start", sid[r], duration_s=dur, active=tools.active_count())
                tel.active_tools += 1
        if done:
            rows = [d.row for d in done]
            nr = [order[r].rounds[rnd[r] + 1] for r in rows]
            c = eng.resume(rows, [d.finish_time for d in done], [d.duration_s for d in done],
                           [x.new_prefill_tokens for x in nr], [x.decode_tokens for x in nr], now)
            for r in rows:
                rnd[r] += 1
            cnt["warm_resumes"] += c["warm"]
            cnt["cold_resumes"] += c["cold"]
            cnt["evictions"] += c["evicted"]
            pinned -= c["warm"] + c["evicted"]
            rr = eng.resume_rows(len(rows)) if (log is not None or tier is not None) else None
            if tier is not None:   # warm resumes: their tables back from the host tier
                tier.after_resume(rows, rr["kind"].tolist(), rr["blocks"].tolist())
            if log is not None:
                for i, d in enumerate(done):
                    r = d.row
                    log.emit(d.finish_time, "tool_end", sid[r], duration_s=d.duration_s,
                             queued_delay_s=d.start_time - d.enqueue_time)
                    tel.active_tools -= 1
                    kind, blk = int(rr["kind"][i]), int(rr["blocks"][i])
                    if kind == 0:
                        log.emit(now, "unpin", sid[r], blocks=blk)
                    elif kind == 2:
                        evict_log(r, blk, "pinned", "pin_expired_at_return", now)
                    proj = int(rr["projected"][i])
                    log.emit(now, "gpu_submit", sid[r], round=rnd[r],
                             required_prefill=int(rr["need"][i]),
                             new_tokens=nr[i].new_prefill_tokens,
                             context_tokens=int(rr["context"][i]), warm=kind == 0,
                             projected_blocks=proj)
                    tel.available_kv -= proj
                    submit_t[r] = now
        # the tick: expiry, probe, control plane, plan, step_gpu, round ends
        due = admission and now >= next_control - 1e-9
        pre = eng.get_scalars() if (log is not None and due) else None
        si = eng.step_in(now, due, tools.active_count(), tools.queued_count(), slots,
                         N.MODE_ADVANCE)
        res = eng.step(si)
        if res.status:
            raise RuntimeError(f"device step status {res.status}")
        if tier is not None:   # evicted / unpinned blocks and new pins to the host tier
            tier.after_step(res)
        if log is not None:
            for r, b in zip(res.expired_rows.tolist(), res.expired_blocks.tolist()):
                evict_log(r, b, "pinned", "pin_expired", now)   # sim.py:324-325
            tel.probe(int(res.free_after_expiry), total_blocks, tools, active)   # sim.py:327
            if due:  # sim.py:328-335: refresh_pressure, telemetry, balance_and_admit
                post = eng.get_scalars()
                post.ema_blocks, post.has_ema_blocks = pre.ema_blocks, pre.has_ema_blocks
                log.emit(now, "telemetry", None, **tel.snapshot(post))
                log.emit(now, "window_update", None, w_adm=float(post.w_adm),
                         limit=int(res.limit), slots=int(res.slots),
                         admitted=[sid[r] for r in res.admitted_rows.tolist()],
                         cpu_overloaded=bool(post.cpu_overloaded),
                         kv_overloaded=bool(post.kv_overloaded))
                for r in res.admitted_rows.tolist():
                    admit_log(r, now)
            # build_plan's ordered pool journal (scheduler.py:300-370 via sim.py:186-188)
            for op, r, k in zip(res.journal_op.tolist(), res.journal_row.tolist(),
                                res.journal_n.tolist()):
                if op == 1:
                    log.emit(now, "alloc", sid[r], blocks=k)
                elif op == 3:
                    evict_log(r, k, "pinned", "reclaim", now)
                else:
                    evict_log(r, k, "running", "preempt", now)
        if due:
            next_control = now + cfg.control_interval_s
            admitted = set(int(x) for x in res.admitted_rows)
            queue = [r for r in queue if r not in admitted]
            cnt["admitted"] += len(admitted)
            active += len(admitted)
        cnt["evictions"] += len(res.expired_rows)
        pinned -= len(res.expired_rows)
        for k in res.evict_kind.tolist():
            cnt["evictions"] += 1
            if k == 0:
                cnt["preemptions"] += 1
            else:
                pinned -= 1
        if res.total_tokens > 0:
            cnt["gpu_tokens"] += int(res.total_tokens)
            end = now + tick
            dec_rows = res.decode_rows.tolist()
            if log is not None:
                log.emit(now, "tick", None, tokens=int(res.total_tokens),
                         decodes=[sid[r] for r in dec_rows],
                         prefills=[[sid[r], g] for r, g in zip(res.prefill_rows.tolist(),
                                                               res.prefill_grants.tolist())],
                         evictions=len(res.evict_rows))
            for e, (r, kind) in enumerate(zip(res.end_rows.tolist(), res.end_kind.tolist())):
                blk = int(res.end_blocks[e])
                if kind == 0:
                    cnt["completed"] += 1
                    active -= 1
                    if log is not None:   # sim.py:240-248
                        if blk > 0:
                            log.emit(end, "free", sid[r], blocks=blk)
                        log.emit(end, "gpu_end", sid[r], round=rnd[r], done=True,
                                 freed_blocks=blk)
                        tel.available_kv += blk
                    continue
                if log is not None and decides:   # sim.py:250-260
                    log.emit(end, "retention", sid[r], pin=bool(res.end_pin[e]),
                             benefit_s=float(res.end_benefit[e]), cost_s=float(res.end_cost[e]),
                             deadline=float(res.end_deadline[e]))
                if kind == 1:
                    cnt["pins"] += 1
                    pinned += 1
                    freed = 0
                    if log is not None:
                        log.emit(end, "pin", sid[r], blocks=blk)
                else:
                    cnt["evictions"] += 1
                    freed = blk
                    if log is not None:
                        if blk > 0:
                            log.emit(end, "free", sid[r], blocks=blk)
                        log.emit(end, "evict", sid[r], blocks=blk, victim="boundary",
                                 reason="tool_boundary")
                dur = order[r].rounds[rnd[r]].tool_duration_s
                dur = dur if dur is not None else 0.0
                if log is not None:
                    log.emit(end, "gpu_end", sid[r], round=rnd[r], done=False, freed_blocks=freed)
                    tel.available_kv += freed
                started = tools.start_tool(r, dur, end)
                if log is not None:   # sim.py:273-279
                    log.emit(end, "tool_num", sid[r], queued=tools.queued_count(), duration_s=dur)
                    if started:
                        log.emit(end, "tool_start", sid[r], duration_s=dur,
                                 active=tools.active_count())
                        tel.active_tools += 1
            if log is not None:   # first tokens (sim.py:365-371), prefills after decodes
                for r, pd in zip(res.prefill_rows.tolist(), res.prefill_done.tolist()):
                    if pd and (r, rnd[r]) not in first_seen:
                        first_seen.add((r, rnd[r]))
                        log.emit(end, "gpu_1st_token", sid[r], round=rnd[r],
                                 launch_delay_s=end - submit_t[r])
            clock = end
            continue
        # idle tick: jump to the next instant anything can change (sim.py:377-418)
        cand = []
        if nxt < n:
            cand.append(order[nxt].arrival_time_s)
        nf = tools.next_finish_time()
        if nf is not None:
            cand.append(nf)
        if admission and (queue or active):
            cand.append(next_control)
        ready = int(res.n_ready) + len(res.admitted_rows) > 0
        if ready or pinned > 0:
            cand.append(now + tick)
        if not cand:
            if active or queue:
                raise RuntimeError("no future event but sessions remain")
            break
        target = min(cand)
        steps = max(1, math.ceil((target - now) / tick - 1e-9))
        clock = now + steps * tick
    if log is not None:   # sim.py:421
        log.emit(clock, "telemetry", None, **tel.snapshot(eng.get_scalars()))
    return cnt, clock
