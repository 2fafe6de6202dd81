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
    if kind == "queue_shuffled":
        # admission list order is persistent state, not row order
        s = snapshot_v1(n, seed=seed, pool="headroom")
        s.queue = np.random.default_rng(seed).permutation(s.queue).astype(np.uint32)
        return partial_admission(s)
    if kind == "queue_sorted":
        # steady state: the residual list is already packed (ascending req),
        # so every range-sort CTA finds its entries in one stretch of the list
        s = snapshot_v1(n, seed=seed, pool="headroom")
        q = s.queue
        s.queue = q[np.argsort(s.cols["req_blocks"][q], kind="stable")].astype(np.uint32)
        return partial_admission(s)
    if kind == "hot_req":
        # a few heavily repeated req values: hot histogram bins (LSD fallback)
        s = snapshot_v1(n, seed=seed, pool="headroom")
        reqs = np.random.default_rng(seed).choice([64, 4096], size=len(s.queue))
        return set_queue_req(s, reqs)
    if kind == "warm_req":
        # five repeated values: each bin spans several range-sort CTAs
        s = snapshot_v1(n, seed=seed, pool="headroom")
        reqs = np.random.default_rng(seed).choice([64, 65, 500, 501, 4096], size=len(s.queue))
        return partial_admission(set_queue_req(s, reqs))
    if kind == "many_equal_req":
        # repeated keys that stay under the hot-bin bound: boundary bins shared
        # by neighbouring range-sort CTAs
        s = snapshot_v1(n, seed=seed, pool="headroom")
        reqs = np.random.default_rng(seed).integers(100, 160, size=len(s.queue))
        return partial_admission(set_queue_req(s, reqs))
    if kind == "wide_req":
        # req_blocks beyond the histogram (LSD fallback), and the largest one
        # a 262144-token context can have
        s = snapshot_v1(n, seed=seed, pool="headroom")
        reqs = s.cols["req_blocks"][s.queue].astype(np.int64)
        reqs[:3] = [16384, 17407, 25000]
        return set_queue_req(s, reqs)
    if kind == "desc_sorted":
        # descending pack (CPU overloaded) of an ascending-sorted list
        s = variant(n, seed, "queue_sorted")
        s.active_tools = s.worker_slots
        s.telemetry = {"cpu_high_streak": 2}
        return partial_admission(s, overloaded=True)
    if kind == "no_queue_control":
        s = snapshot_v1(n, seed=seed, pool="headroom")
        q = s.queue
        s.cols["flags"][q] &= ~np.uint8(F_QUEUED)
        s.cols["phase"][q] = 5
        s.queue = q[:0]
        return s
    raise ValueError(kind)


def set_queue_req(snap, reqs):
    """Give the queued sessions new first-round prefills (req_blocks = reqs)."""
    q = snap.queue
    reqs = np.asarray(reqs, dtype=np.int64)
    snap.cols["req_blocks"][q] = reqs
    snap.cols["r0_prefill"][q] = reqs * 16 - 3
    long_ = reqs > 0.25 * snap.total_blocks
    snap.cols["flags"][q] = (snap.cols["flags"][q] & ~np.uint8(F_LONG)) | np.where(
        long_, F_LONG, 0).astype(np.uint8)
    return snap


def partial_admission(snap, overloaded=False):
    """Admission window so that about a third of the list is admitted: the
    residual list order (persistent state, control.py:190) is then checked."""
    active = int(((snap.cols["flags"] & 1) != 0).sum())
    w = active + len(snap.queue) // 3
    snap.initial_window = float(2 * w if overloaded else w)  # AIMD halves it under overload
    return snap


def comparison_variant(n, seed, policy, pool):
    """A snapshot the reference's comparison policies can hold: fcfs and
    program_priority never pin (their pinned rows become unpinned tool rows
    and the pool shrinks by those blocks, so the pressure is unchanged);
    program_priority's `served` column is Call.served_tokens, with ties and
    small values so every branch of its key and digit runs."""
    s = snapshot_v1(n, seed=seed, pool=pool)
    c = s.cols
    rng = np.random.default_rng(seed + 1000)
    if policy in ("fcfs", "program_priority"):
        pinned = (c["flags"] & F_PINNED) != 0
        blocks = int(c["pinned_blocks"][pinned].astype(np.int64).sum())
        c["flags"][pinned] &= ~np.uint8(F_PINNED)
        c["kv"][pinned] = 0
        c["pinned_blocks"][pinned] = 0
        c["deadline"][pinned] = 0.0
        c["plevel"][pinned] = 0
        s.total_blocks -= blocks
    if policy == "program_priority":
        served = rng.integers(0, 60_000, size=n)
        u = rng.random(n)
        served[u < 0.05] = 0
        served[(u >= 0.05) & (u < 0.08)] = rng.integers(1, 8, size=int(((u >= 0.05) & (u < 0.08)).sum()))
        served[(u >= 0.08) & (u < 0.10)] = 4096
        c["served"][:] = served
    return s


def tick_grid(snap, seed, tick=0.064, batch_frac=0.05):
    """Times on the reference clock's tick grid (engine.py:71-74: the clock
    advances by repeated `now + tick_duration`), so ready_since / wait_since /
    arrival tie exactly across many sessions, and a batch of sessions admitted
    together shares ready_since == now (sim.py:148-166)."""
    c = snap.cols
    n = snap.n
    rng = np.random.default_rng(seed + 4242)
    k_now = int(round(snap.now / tick))
    grid = np.cumsum(np.full(k_now + 400, tick))          # sequential IEEE adds
    now = float(grid[k_now - 1])
    ir = rng.integers(0, k_now, size=n)
    ir[rng.random(n) < batch_frac] = k_now - 1              # admitted at `now` together
    iw = np.minimum(ir + rng.integers(0, 313, size=n), k_now - 1)
    ia = (ir * rng.random(n)).astype(np.int64)
    c["ready_since"][:] = grid[ir]
    c["wait_since"][:] = grid[iw]
    c["arrival"][:] = grid[ia]
    pinned = (c["flags"] & F_PINNED) != 0
    c["deadline"][pinned] += now - snap.now
    snap.now = now
    snap.meta = dict(snap.meta, tick_grid=True)
    return snap


def reclaim_heavy(n, seed, policy="mars", tiny_pins=40):
    """A step that needs many victims (scheduler.py:228-267 returning long
    prefixes): every running session holds 1-2 blocks, decodes are block
    aligned (each needs one new block), prefills are whole chunks from a
    block-aligned KV, and the pool has no free block.  Policies that pin keep
    a few one-block pins (reclaimed first); fcfs / program_priority hold none."""
    from paper_2604_26963_b200.snapshot import DECODE, PREFILL

    s = snapshot_v1(n, seed=seed, pool="pressure")
    c = s.cols
    rng = np.random.default_rng(seed + 99)
    dec = c["phase"] == DECODE
    pre = c["phase"] == PREFILL
    small = 16 * rng.integers(1, 3, size=n)
    c["kv"][dec] = small[dec]
    c["context"][dec] = small[dec]
    c["kv"][pre] = 16 * rng.integers(0, 2, size=n)[pre]
    pinned = (c["flags"] & F_PINNED) != 0
    keep = np.zeros(n, dtype=bool)
    if policy not in ("fcfs", "program_priority"):
        keep[rng.permutation(np.nonzero(pinned)[0])[:tiny_pins]] = True
    drop = pinned & ~keep
    c["flags"][drop] &= ~np.uint8(F_PINNED)
    c["kv"][drop] = 0
    c["pinned_blocks"][drop] = 0
    c["deadline"][drop] = 0.0
    c["plevel"][drop] = 0
    c["kv"][keep] = 16
    c["pinned_blocks"][keep] = 1
    held = -(-c["kv"].astype(np.int64) // 16)
    s.total_blocks = int(held.sum())
    s.free_blocks = 0
    q = s.queue
    long_ = c["req_blocks"][q] > 0.25 * s.total_blocks
    c["flags"][q] = (c["flags"][q] & ~np.uint8(F_LONG)) | np.where(long_, F_LONG, 0).astype(np.uint8)
    if policy == "program_priority":
        served = rng.integers(0, 60_000, size=n)
        u = rng.random(n)
        served[u < 0.05] = 0
        served[(u >= 0.05) & (u < 0.10)] = 4096
        c["served"][:] = served
    s.meta = dict(s.meta, variant="reclaim_heavy", policy=policy)
    return s


def kv_small(n, seed):
    """The headroom mix with small KV footprints (1-4 blocks per session), so
    the CPU block-ID restatement (oracle/block_ids.py) can follow a 1M-session
    table: running and pinned sessions hold 16-64 tokens, prefills 0-63, the
    pool keeps the headroom rule and ~8% of the pins expire this step."""
    from paper_2604_26963_b200.snapshot import DECODE, PREFILL

    s = snapshot_v1(n, seed=seed, pool="headroom")
    c = s.cols
    rng = np.random.default_rng(seed + 5)
    dec = c["phase"] == DECODE
    pre = c["phase"] == PREFILL
    pinned = (c["flags"] & F_PINNED) != 0
    small = 16 * rng.integers(1, 5, size=n)
    c["kv"][dec | pinned] = small[dec | pinned]
    c["context"][dec] = small[dec]
    c["kv"][pre] = rng.integers(0, 64, size=n)[pre]
    c["pinned_blocks"][pinned] = small[pinned] // 16
    held = np.where(pinned, c["pinned_blocks"], -(-c["kv"].astype(np.int64) // 16))
    total_held = int(held.sum())
    s.total_blocks = -(-total_held * 100 // 85)
    s.free_blocks = s.total_blocks - total_held
    q = s.queue
    long_ = c["req_blocks"][q] > 0.25 * s.total_blocks
    c["flags"][q] = (c["flags"][q] & ~np.uint8(F_LONG)) | np.where(long_, F_LONG, 0).astype(np.uint8)
    s.meta = dict(s.meta, variant="kv_small")
    return s
