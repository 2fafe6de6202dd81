"""Seeded synthetic session-table snapshots (``snapshot_v1``).

A snapshot is the structure-of-arrays session table the B200 step runs over,
plus the scalar state around it (pool, telemetry, controller, tool plane).
It is plain numpy so the same arrays feed the device upload and the CPU
oracle.  Column meanings mirror the reference's per-session state:

* ``Call`` (agentsched/engine.py:259-289): phase, context, kv, rem_decode,
  ready_since, arrival, preempt, the current round's new-prefill / decode
  lengths (r0_prefill / r0_decode).
* ``PriorityState`` (scheduler.py:78-84): level, promos, wait_since, served.
* ``PinnedSession`` (scheduler.py:165-172): deadline, pinned_blocks, plevel.
* ``QueueEntry`` (control.py:64-73): req_blocks, the LONG flag; the list
  order is the separate ``queue`` row-index array.
* ``rank``: dense rank of the session-id string in lexicographic order, the
  reference's final tie-break (baselines.py:374-377).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, Optional

import numpy as np

# phase codes (agentsched/engine.py:250-256 order)
WAITING_ADMISSION, PREFILL, DECODE, TOOL, WAITING_RESUME, DONE, EMPTY = 0, 1, 2, 3, 4, 5, 7
PHASE_NAMES = ("waiting_admission", "prefill", "decode", "tool", "waiting_resume", "done")

# flag bits
F_ACTIVE, F_QUEUED, F_PINNED, F_BOUNDARY, F_LONG = 1, 2, 4, 8, 16

BLOCK = 16
LEVEL_BOUNDS = (4_000, 32_000, 128_000)

COLUMNS = {
    "phase": np.uint8, "flags": np.uint8, "level": np.uint8, "promos": np.uint8,
    "plevel": np.uint8,
    "ready_since": np.float64, "wait_since": np.float64, "deadline": np.float64,
    "arrival": np.float64,
    "context": np.int32, "kv": np.int32, "rem_decode": np.int32, "pinned_blocks": np.int32,
    "req_blocks": np.int32, "r0_prefill": np.int32, "r0_decode": np.int32,
    "preempt": np.int32, "served": np.int64, "rank": np.uint32, "rounds_left": np.int32,
}


@dataclass
class Snapshot:
    cols: Dict[str, np.ndarray]
    queue: np.ndarray                 # u32 row ids in admission-list order
    now: float
    total_blocks: int
    free_blocks: int
    worker_slots: int
    active_tools: int
    queued_tools: int
    initial_window: float
    ema_tool: Optional[float] = 5.0
    ema_blocks: Optional[float] = None
    blocks_seed: Optional[float] = None
    # initial Telemetry hysteresis state (telemetry.py:80-91): any of
    # cpu_overloaded, kv_overloaded, cpu_high_streak, cpu_low_streak,
    # kv_high_streak, kv_low_streak
    telemetry: dict = field(default_factory=dict)
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.cols["phase"].shape[0])

    def sid(self, row: int) -> str:
        return sid_of(int(self.cols["rank"][row]))

    def copy(self) -> "Snapshot":
        s = Snapshot(**{k: getattr(self, k) for k in self.__dataclass_fields__})
        s.cols = {k: v.copy() for k, v in self.cols.items()}
        s.queue = self.queue.copy()
        s.meta = dict(self.meta)
        s.telemetry = dict(self.telemetry)
        return s


def sid_of(rank: int) -> str:
    """Session ids ``s0000000``..: fixed width, so lexicographic rank == i."""
    return f"s{rank:07d}"


def initial_level_np(tokens: np.ndarray) -> np.ndarray:
    """initial_level (scheduler.py:87-97) for the default boundaries."""
    lv = np.full(tokens.shape, 3, dtype=np.uint8)
    for i, b in reversed(list(enumerate(LEVEL_BOUNDS))):
        lv[tokens <= b] = i
    return lv


def snapshot_v1(n: int, seed: int = 0, pool: str = "headroom", now: float = 1000.0) -> Snapshot:
    """Mix-A snapshot: 50% DECODE, 25% PREFILL, 15% TOOL (60% pinned), 10% queued.

    ``pool="headroom"``: total = ceil(sum(held) / 0.85); pins expire with
    p = 5/65 (deadline = now + U(-5, 60)).  ``pool="pressure"``: total =
    sum(held) + 8 and no pin has expired (deadline = now + U(0, 60)], so
    chunk fitting fails and reclamation runs.
    """
    if pool not in ("headroom", "pressure"):
        raise ValueError(pool)
    rng = np.random.Generator(np.random.PCG64(seed))
    c = {k: np.zeros(n, dtype=t) for k, t in COLUMNS.items()}
    ctx = np.rint(1000.0 * 128.0 ** rng.random(n)).astype(np.int64)
    u = rng.random(n)
    phase = np.where(u < 0.50, DECODE, np.where(u < 0.75, PREFILL,
                     np.where(u < 0.90, TOOL, WAITING_ADMISSION))).astype(np.uint8)
    dec = phase == DECODE
    pre = phase == PREFILL
    tool = phase == TOOL
    waiting = phase == WAITING_ADMISSION
    pinned = tool & (rng.random(n) < 0.6)
    kv_pre = (rng.random(n) * ctx).astype(np.int64)           # U{0..ctx-1}
    kv = np.where(dec | pinned, ctx, np.where(pre, kv_pre, 0))
    rem = rng.integers(1, 65, size=n)
    if pool == "headroom":
        dl = now + rng.uniform(-5.0, 60.0, size=n)
    else:
        dl = now + 60.0 * (1.0 - rng.random(n))                # (0, 60]
    lvl = initial_level_np(ctx)
    demote = rng.random(n) < 0.3
    lvl = np.minimum(lvl + demote, 3).astype(np.uint8)
    promos = rng.integers(0, 4, size=n).astype(np.uint8)
    rs = rng.uniform(0.0, now, size=n)
    ws = np.minimum(now, rs + rng.uniform(0.0, 20.0, size=n))
    arr = rs * rng.random(n)
    boundary = dec & (rng.random(n) < 1.0 / 16.0)

    c["phase"][:] = phase
    c["context"][:] = np.where(waiting, 0, ctx)
    c["kv"][:] = kv
    c["rem_decode"][:] = np.where(dec, rem, 0)
    c["r0_prefill"][:] = np.where(waiting, ctx, 0)
    c["r0_decode"][:] = np.where(waiting, rem, 0)
    c["req_blocks"][:] = np.where(waiting, -(-ctx // BLOCK), 0)
    c["level"][:] = lvl
    c["promos"][:] = promos
    c["ready_since"][:] = rs
    c["wait_since"][:] = ws
    c["arrival"][:] = arr
    c["deadline"][:] = np.where(pinned, dl, 0.0)
    held = -(-kv // BLOCK)
    c["pinned_blocks"][:] = np.where(pinned, held, 0)
    c["plevel"][:] = np.where(pinned, lvl, 0)
    c["rank"][:] = np.arange(n, dtype=np.uint32)
    total_held = int(held.sum())
    total = -(-total_held * 100 // 85) if pool == "headroom" else total_held + 8
    total = max(total, 1)
    long_ = c["req_blocks"] > 0.25 * total
    flags = np.zeros(n, dtype=np.uint8)
    flags |= np.where(dec | pre | tool, F_ACTIVE, 0).astype(np.uint8)
    flags |= np.where(waiting, F_QUEUED, 0).astype(np.uint8)
    flags |= np.where(pinned, F_PINNED, 0).astype(np.uint8)
    flags |= np.where(boundary, F_BOUNDARY, 0).astype(np.uint8)
    flags |= np.where(waiting & long_, F_LONG, 0).astype(np.uint8)
    c["flags"][:] = flags
    queue = np.nonzero(waiting)[0].astype(np.uint32)
    # rounds after the current one (drawn last: the other columns keep their values)
    c["rounds_left"][:] = rng.integers(0, 4, size=n)
    return Snapshot(cols=c, queue=queue, now=float(now), total_blocks=int(total),
                    free_blocks=int(total - total_held), worker_slots=max(2 * n, 1),
                    active_tools=int(tool.sum()), queued_tools=0,
                    initial_window=float(max(2 * n, 8)),
                    meta={"kind": "snapshot_v1", "n": n, "seed": seed, "pool": pool, "mix": "A"})


def snapshot_shard(snap: Snapshot, G: int, g: int, box_global: bool = False) -> Snapshot:
    """Row shard ``g`` of ``G`` (rows ``r`` with ``r % G == g``, SURVEY.md
    §8(e): session row -> replica ``sid_rank mod G``; ``snapshot_v1`` ranks
    equal rows).  Its rows keep their session ids (rank), its pool holds its
    own rows' blocks with the same headroom rule (or the same +8 slack under
    pressure), its admission list is its rows in the global list order, and
    ``meta["gpos"]`` holds each of those entries' position in the global list.

    ``box_global=False``: the shard is an independent replica (the tool plane
    and admission window scale with its size).  ``box_global=True``: one
    replica of a sharded engine (config 3): the tool-plane counters, worker
    slots and the admission window stay the box's (identical on every rank),
    as the sharded control plane sees them (oracle/multi.py)."""
    if not (0 <= g < G):
        raise ValueError((G, g))
    rows = np.arange(g, snap.n, G)
    c = {k: v[rows].copy() for k, v in snap.cols.items()}
    n = len(rows)
    held = -(-c["kv"].astype(np.int64) // BLOCK)
    total_held = int(held.sum())
    pool = snap.meta.get("pool", "headroom")
    slack = snap.total_blocks - (snap.total_blocks - snap.free_blocks)
    if pool == "headroom":
        total = -(-total_held * 100 // 85)
    else:
        total = total_held + min(slack, 8)
    total = max(total, 1)
    q = snap.queue[snap.queue % G == g]
    queue = (q // G).astype(np.uint32)
    long_ = c["req_blocks"] > 0.25 * total
    fl = c["flags"]
    waiting = (fl & F_QUEUED) != 0
    c["flags"][:] = (fl & ~np.uint8(F_LONG)) | np.where(waiting & long_, F_LONG, 0).astype(np.uint8)
    meta = dict(snap.meta, shard=(G, g), n=n,
                gpos=np.nonzero(snap.queue % G == g)[0].astype(np.uint32))
    if box_global:
        slots, tools, qtools, win = (snap.worker_slots, snap.active_tools, snap.queued_tools,
                                     snap.initial_window)
    else:
        slots, tools, qtools, win = (max(2 * n, 1), int((c["phase"] == TOOL).sum()), 0,
                                     float(max(2 * n, 8)))
    return Snapshot(cols=c, queue=queue, now=snap.now, total_blocks=int(total),
                    free_blocks=int(total - total_held), worker_slots=slots,
                    active_tools=tools, queued_tools=qtools,
                    initial_window=win, ema_tool=snap.ema_tool,
                    ema_blocks=snap.ema_blocks, blocks_seed=snap.blocks_seed,
                    telemetry=dict(snap.telemetry), meta=meta)
