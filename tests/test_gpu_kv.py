"""S5 on the B200: block-ID manager parity with the CPU restatement
(oracle/block_ids.py) and exact KV byte round trips through the host tier."""

import random

import numpy as np
import pytest

from oracle.block_ids import BlockIdPool
from oracle.snapshot_step import run_step
from paper_2604_26963_b200 import _native as N
from paper_2604_26963_b200.engine import MarsEngine, make_config
from paper_2604_26963_b200.kvstore import KvBlockManager, host_link_peak
from paper_2604_26963_b200.policy import GpuMarsPolicy
from paper_2604_26963_b200.snapshot import F_PINNED, snapshot_v1
from paper_2604_26963_b200.admission import balance_and_admit
from tests._sim import run_sim

pytestmark = pytest.mark.gpu


def _same_state(kv, pool: BlockIdPool, rows):
    for sid, r in rows.items():
        assert kv.table(r).tolist() == pool.table(sid), sid
    top, depth, fresh, status = kv.state(64)
    assert status == 0
    assert top.tolist() == pool.top(64)
    assert depth + (pool.total - fresh) == len(pool.stack)


def test_fuzzed_op_stream_matches_the_restatement():
    # acceptance criterion 3's op mix (test_acceptance.py:334-366) on block IDs
    rng = random.Random(303)
    total = 512
    eng = MarsEngine(max_rows=32768, max_queue=1)
    kv = KvBlockManager(eng, total, max_blocks_per_row=total)
    ref = BlockIdPool(total)
    alloc, pinned, rows = {}, {}, {}
    ops = []
    for step in range(100_000):
        choices = ["alloc_new"]
        if alloc:
            choices += ["alloc_more", "free_some", "free_all", "pin"]
        if pinned:
            choices += ["unpin", "release_pinned"]
        op = rng.choice(choices)
        free_now = total - sum(alloc.values()) - sum(pinned.values())
        if op in ("alloc_new", "alloc_more"):
            n = rng.randrange(1, 48)
            if n > free_now:
                continue
            sid = f"f{len(rows)}" if op == "alloc_new" else rng.choice(sorted(alloc))
            rows.setdefault(sid, len(rows))
            alloc[sid] = alloc.get(sid, 0) + n
            ref.apply("alloc", sid, n)
            ops.append((N.KV_ALLOC, rows[sid], n))
        elif op in ("free_some", "free_all"):
            sid = rng.choice(sorted(alloc))
            n = rng.randrange(1, alloc[sid] + 1) if op == "free_some" else alloc[sid]
            alloc[sid] -= n
            if not alloc[sid]:
                del alloc[sid]
            ref.apply("free", sid, n)
            ops.append((N.KV_FREE, rows[sid], n))
        elif op == "pin":
            sid = rng.choice(sorted(alloc))
            pinned[sid] = alloc.pop(sid)
            ops.append((N.KV_PIN, rows[sid], pinned[sid]))
        elif op == "unpin":
            sid = rng.choice(sorted(pinned))
            alloc[sid] = pinned.pop(sid)
            ops.append((N.KV_UNPIN, rows[sid], alloc[sid]))
        else:
            sid = rng.choice(sorted(pinned))
            n = pinned.pop(sid)
            ref.apply("free", sid, n)
            ops.append((N.KV_FREE, rows[sid], n))
        if len(ops) >= 2_000:
            kv.apply(ops)
            ops = []
            _same_state(kv, ref, {s: r for s, r in rows.items() if s in ref.tables})
    kv.apply(ops)
    _same_state(kv, ref, rows)
    eng.close()


def test_step_journal_updates_block_tables_like_the_restatement():
    snap = snapshot_v1(20_000, seed=51, pool="pressure")
    c = snap.cols
    eng = MarsEngine(max_rows=snap.n, max_queue=len(snap.queue),
                     config=make_config(initial_window=snap.initial_window))
    eng.load_snapshot(snap)
    kv = KvBlockManager(eng, snap.total_blocks, max_blocks_per_row=1 << 14)
    ref = BlockIdPool(snap.total_blocks)
    held = -(-c["kv"].astype(np.int64) // 16)
    init = []
    for r in range(snap.n):
        h = int(c["pinned_blocks"][r]) if c["flags"][r] & F_PINNED else int(held[r])
        if h:
            init.append((N.KV_ALLOC, r, h))
            ref.apply("alloc", snap.sid(r), h)
    kv.apply(init)
    res = eng.step(eng.step_in(snap.now, True, snap.active_tools, 0, snap.worker_slots))
    assert res.status == 0
    out = run_step(snap.copy())
    assert len(out["evictions"]) > 0
    for op, r, n, from_pinned in out["expiry_journal"] + out["journal"]:
        ref.apply(op, snap.sid(r), n)
    touched = {snap.sid(r) for _, r, _, _ in out["expiry_journal"] + out["journal"]}
    _same_state(kv, ref, {s: int(s[1:]) for s in touched})
    eng.close()


@pytest.mark.parametrize("method", [0, 1, 2])
def test_kv_bytes_round_trip_through_the_host_tier(method):
    bb, layers = 2 << 20, 32
    eng = MarsEngine(max_rows=64, max_queue=1)
    kv = KvBlockManager(eng, 256, max_blocks_per_row=256, block_bytes=bb, layers=layers,
                        host_blocks=64)
    host = kv.host_view()
    rng = np.random.default_rng(7)
    host[:16] = rng.integers(0, 256, size=(16, bb), dtype=np.uint8)
    src = host[:16].copy()
    ids = rng.choice(256, size=16, replace=False).astype(np.uint32)
    kv.restore(ids, slot0=0, method=method)        # host slots 0..15 -> scattered blocks
    host[:16] = 0
    kv.evict(ids, slot0=32, method=method)         # blocks -> host slots 32..47
    assert np.array_equal(host[32:48], src)
    # per-block checksums survive a second scattered hop
    ids2 = rng.choice(256, size=16, replace=False).astype(np.uint32)
    kv.restore(ids2, slot0=32, method=(method + 1) % 3)
    kv.evict(ids2, slot0=0, method=method)
    assert [int(x) for x in host[:16].sum(axis=1, dtype=np.uint64)] == \
        [int(x) for x in src.sum(axis=1, dtype=np.uint64)]
    eng.close()


def test_host_link_peak_is_measurable():
    eng = MarsEngine(max_rows=16, max_queue=1)
    d2h, h2d, bi = host_link_peak(eng, 1 << 28, 3)
    eng.close()
    assert d2h > 1.0 and h2d > 1.0 and bi > 1.0


@pytest.mark.parametrize("key", ["demo64/mars", "faceoff200/mars"])
def test_dropin_block_ids_follow_the_reference_op_stream(key):
    """Drop-in run with the device block manager teed onto the pool: the log
    stays byte-identical and the final tables equal the restatement replaying
    the reference's own pool op stream."""
    import hashlib

    from tests._sim import SIM

    pol = GpuMarsPolicy(kv_blocks=True)
    out = run_sim(key, policy=pol, balance_and_admit=balance_and_admit)
    pol.kv_flush()
    assert hashlib.sha256(out.log.jsonl_bytes()).hexdigest() == SIM[key]["sha256"]
    ref = BlockIdPool(out.pool.total_blocks)
    for rec in out.events:
        if rec["kind"] in ("alloc", "free", "pin", "unpin"):
            ref.apply(rec["kind"], rec["session_id"], rec["blocks"])
    rows = {sid: pol._row[sid] for sid in pol._row}
    _same_state(pol.kv, ref, rows)
    pol.close()


def _ref_tables(snap):
    """The restatement holding every session's initial table: sequential
    allocs in session-id order (what mars_kv_bulk_alloc reproduces)."""
    c = snap.cols
    held = -(-c["kv"].astype(np.int64) // 16)
    blocks = np.where((c["flags"] & F_PINNED) != 0, c["pinned_blocks"], held)
    ref = BlockIdPool(snap.total_blocks)
    for r in np.argsort(c["rank"], kind="stable"):
        if blocks[r] > 0:
            ref.apply("alloc", snap.sid(int(r)), int(blocks[r]))
    return ref


def test_bulk_alloc_matches_sequential_allocs():
    from tests._variants import kv_small
    snap = kv_small(30_000, 61)
    eng = MarsEngine(max_rows=snap.n, max_queue=len(snap.queue),
                     config=make_config(initial_window=snap.initial_window))
    eng.load_snapshot(snap)
    kv = KvBlockManager(eng, snap.total_blocks, max_blocks_per_row=1 << 10)
    kv.load_snapshot_tables(snap)
    ref = _ref_tables(snap)
    rows = {snap.sid(r): r for r in range(0, snap.n, 97)}
    _same_state(kv, ref, {s: r for s, r in rows.items() if s in ref.tables})
    eng.close()


@pytest.mark.parametrize("n,kind", [(1_000_000, "kv_small"), (200_000, "reclaim_heavy"),
                                    (100_000, "pressure_small")])
def test_step_with_block_ids_at_scale_matches_the_restatement(n, kind):
    """The whole step with S5 attached (expired pins' tables back on the stack
    grid-wide, then the plan's alloc / evict journal) against the
    restatement replaying the oracle's op stream."""
    from tests._variants import kv_small, reclaim_heavy, with_free
    if kind == "kv_small":
        snap = kv_small(n, 62)
    elif kind == "reclaim_heavy":
        snap = reclaim_heavy(n, 63, "mars")
    else:
        snap = with_free(kv_small(n, 64), 3)
    eng = MarsEngine(max_rows=snap.n, max_queue=len(snap.queue),
                     config=make_config(initial_window=snap.initial_window))
    eng.load_snapshot(snap)
    kv = KvBlockManager(eng, snap.total_blocks, max_blocks_per_row=1 << 10)
    kv.load_snapshot_tables(snap)
    eng.set_graph(True)
    res = eng.step(eng.step_in(snap.now, True, snap.active_tools, 0, snap.worker_slots))
    assert res.status == 0
    ref = _ref_tables(snap)
    out = run_step(snap.copy())
    for op, r, k, from_pinned in out["expiry_journal"] + out["journal"]:
        ref.apply(op, snap.sid(r), k)
    touched = {snap.sid(r) for _, r, _, _ in out["expiry_journal"] + out["journal"]}
    assert touched
    _same_state(kv, ref, {s: int(s[1:]) for s in touched if int(s[1:]) < snap.n})
    top, depth, fresh, status = kv.state(4096)
    assert top.tolist() == ref.top(4096)
    eng.close()


def test_deep_alloc_run_pops_many_small_segments():
    """An alloc popping more than 1024 one-ID segments at once (the
    sequential fallback of the run kernel)."""
    eng = MarsEngine(max_rows=4096, max_queue=1)
    total = 8192
    kv = KvBlockManager(eng, total, max_blocks_per_row=4096)
    ref = BlockIdPool(total)
    ops = []
    for r in range(3000):
        ops.append((N.KV_ALLOC, r, 2))
        ref.apply("alloc", f"s{r}", 2)
    for r in range(3000):
        ops.append((N.KV_FREE, r, 1))
        ref.apply("free", f"s{r}", 1)
    ops.append((N.KV_ALLOC, 3500, 2500))
    ref.apply("alloc", "s3500", 2500)
    kv.apply(ops)
    _same_state(kv, ref, {"s3500": 3500, "s17": 17, "s2999": 2999})
    eng.close()


@pytest.mark.parametrize("key", ["openhands_heavy40/mars", "demo64/mars", "small12/mars-no-coscheduler"])
def test_host_tier_follows_the_decisions(key):
    """the KV bytes move as the run's decisions imply
    -- a pin copies the table to the host ring, a warm resume copies it back,
    a running session's eviction and an unpinned tool boundary copy the freed
    blocks out (captured on the device while the step frees them) -- while
    the event log stays the reference's byte for byte.  Every host slot holds
    the block it was given and no pool block is corrupted by the restores."""
    from oracle import tracefile
    from paper_2604_26963_b200.devsim import EventLog, run_device_simulation
    from tests._sim import SIM, VARIANT_KW
    from tests.conftest import GOLDEN
    import hashlib
    import os
    spec = SIM[key]
    traces = tracefile.load(os.path.join(GOLDEN, spec["trace"]))
    log, kv = EventLog(), {}
    tier = {"block_bytes": 1024, "pattern": True, "verify": True}
    run_device_simulation(traces, spec["engine"]["total_blocks"], spec["engine"]["tool_worker_slots"],
                          enable_control_plane=spec["run"].get("enable_control_plane", True),
                          log=log, kv_state=kv, kv_tier=tier, **VARIANT_KW[key.split("/")[1]])
    assert hashlib.sha256(log.jsonl_bytes()).hexdigest() == spec["sha256"]
    assert kv["status"] == 0
    recs = log.records
    out = sum(r["blocks"] for r in recs if r["kind"] == "evict" and r["victim"] in ("running", "boundary"))
    assert tier["evict_blocks"] == out
    assert tier["pin_blocks"] == sum(r["blocks"] for r in recs if r["kind"] == "pin")
    assert tier["restore_blocks"] == sum(r["blocks"] for r in recs if r["kind"] == "unpin")
    assert tier["evict_blocks"] + tier["pin_blocks"] > 0
    assert tier["host_slots_checked"] > 0 and tier["host_slots_bad"] == 0
    assert tier["pool_blocks_bad"] == 0


def test_batched_hooks_larger_than_the_staging_buffer():
    """mars_on_admit / mars_queue_append take batches of any size (passed
    through the row staging buffer in chunks)."""
    from paper_2604_26963_b200.snapshot import initial_level_np
    n = 2000
    eng = MarsEngine(max_rows=n, max_queue=n)
    rng = np.random.default_rng(3)
    rows = rng.permutation(n)[:1900].astype(np.int64)
    r0 = rng.integers(1, 200_000, size=len(rows)).astype(np.int32)
    eng.upsert({"level": np.full(n, 9, np.uint8), "promos": np.full(n, 2, np.uint8),
                "served": np.full(n, 7, np.int64), "flags": np.zeros(n, np.uint8)})
    eng.on_admit(rows, r0, 12.5)
    st = eng.read(["level", "promos", "served", "wait_since", "flags"], rows=rows)
    assert st["level"].tolist() == initial_level_np(r0.astype(np.int64)).tolist()
    assert not st["promos"].any() and not st["served"].any()
    assert (st["wait_since"] == 12.5).all() and (st["flags"] & 1).all()
    q = rng.permutation(n)[:1800].astype(np.uint32)
    req = rng.integers(1, 500, size=len(q)).astype(np.int32)
    eng.set_queue(q[:5], req[:5], np.zeros(5, bool))
    eng.queue_append(q[5:], req[5:], np.zeros(len(q) - 5, bool))
    assert eng.get_queue().tolist() == q.tolist()
    eng.close()
