"""Snapshot variants that drive every branch of the step (shared by tests)."""

import numpy as np

from paper_2604_26963_b200.snapshot import F_LONG, F_PINNED, F_QUEUED, snapshot_v1


def with_free(snap, free):
    used = snap.total_blocks - snap.free_blocks
    snap.total_blocks = used + int(free)
    snap.free_blocks = int(free)
    return snap


def variant(n, seed, kind):
    if kind in ("headroom", "pressure"):
        return snapshot_v1(n, seed=seed, pool=kind)
    if kind == "first_fit":
        s = snapshot_v1(n, seed=seed, pool="pressure")
        q = s.queue
        s.cols["flags"][q] |= F_LONG
        reqs = np.sort(s.cols["req_blocks"][q])
        return with_free(s, int(reqs[: max(1, len(reqs) // 5)].sum()))
    if kind == "desc":
        s = snapshot_v1(n, seed=seed, pool="headroom")
        s.active_tools = s.worker_slots
        s.telemetry = {"cpu_high_streak": 2}
        return s
    if kind == "expired_big":
        s = snapshot_v1(n, seed=seed, pool="headroom")
        pinned = (s.cols["flags"] & F_PINNED) != 0
        s.cols["deadline"][pinned] = s.now - 1.0
        return s
    if kind == "expired_shuffled":
        # session ids not in row order: the expired pins need the rank sort
        # (> 4096 of them: the grid-wide LSD path)
        s = variant(n, seed, "expired_big")
        s.cols["rank"][:] = np.random.default_rng(seed).permutation(n).astype(np.uint32)
        return s
    if kind == "no_queue_control":
        s = snapshot_v1(n, seed=seed, pool="headroom")
        q = s.queue
        s.cols["flags"][q] &= ~np.uint8(F_QUEUED)
        s.cols["phase"][q] = 5
        s.queue = q[:0]
        return s
    raise ValueError(kind)
