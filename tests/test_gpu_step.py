"""Parity of the B200 step (through the C ABI) with the reference.

* small snapshots: against outputs frozen from the reference itself
  (tests/golden/snapshot_steps.json);
* up to 1M sessions: against the CPU oracle on the same seeded inputs,
  every decision bit-exact (window, plan, evictions, journal, expiry order,
  admitted set + residual queue order, retention f64 values) plus the full
  post-step session table.
"""

import json
import os

import numpy as np
import pytest

from oracle.snapshot_step import run_step
from paper_2604_26963_b200.engine import MarsEngine, canonical, make_config
from paper_2604_26963_b200.snapshot import snapshot_v1
from tests._canon import canon
from tests._variants import comparison_variant, variant
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

SNAP = json.load(open(os.path.join(GOLDEN, "snapshot_steps.json")))


def device_step(snap, control_due=True, sort_path=None, **flags):
    eng = MarsEngine(max_rows=snap.n, max_queue=max(len(snap.queue), 1),
                     config=make_config(**flags, initial_window=snap.initial_window))
    eng.load_snapshot(snap)
    si = eng.step_in(snap.now, control_due, snap.active_tools, snap.queued_tools,
                     snap.worker_slots)
    res = eng.step(si)
    out = canonical(res, eng, snap, control_due)
    eng.close()
    assert res.status == 0, res.status
    if sort_path is not None:
        assert res.diag["sort_path"] == sort_path, res.diag
    return out


def assert_same(got, want):
    g, w = canon(got), canon(want)
    for k in w:
        if g[k] != w[k]:
            gs, ws = json.dumps(g[k]), json.dumps(w[k])
            raise AssertionError(f"{k} differs:\n device {gs[:600]}\n oracle {ws[:600]}")


@pytest.mark.parametrize("i", range(len(SNAP)))
def test_step_matches_reference_golden(i):
    case = dict(SNAP[i]["case"])
    kw = {k: case.pop(k) for k in ("enable_coordinator", "enable_coscheduler") if k in case}
    snap = snapshot_v1(case["n"], seed=case["seed"], pool=case["pool"])
    got = canon(device_step(snap, **kw))
    for k, v in SNAP[i]["out"].items():
        assert got[k] == v, k


# how pack_queue's sort must run: 3 grid-wide LSD radix sort concurrently with
# the table scan (k_pack, big list), 1 the same inside the control plane, 2
# one CTA (small list, or the first-fit mode)
SORT_PATH = {"headroom": 3, "pressure": 3, "first_fit": 2, "desc": 2, "queue_shuffled": 3,
             "queue_sorted": 3, "hot_req": 3, "many_equal_req": 3, "warm_req": 3,
             "wide_req": 3, "desc_sorted": 3}


@pytest.mark.parametrize("n,seed,kind", [
    (100_000, 21, "headroom"),
    (100_000, 22, "pressure"),
    (30_000, 23, "first_fit"),
    (30_000, 24, "desc"),
    (150_000, 25, "expired_big"),
    (150_000, 27, "expired_shuffled"),
    (20_000, 26, "no_queue_control"),
    (200_000, 28, "queue_shuffled"),
    (200_000, 29, "queue_sorted"),
    (100_000, 30, "hot_req"),
    (100_000, 33, "many_equal_req"),
    (100_000, 36, "warm_req"),
    (60_000, 34, "wide_req"),
    (60_000, 35, "desc_sorted"),
])
def test_step_matches_oracle(n, seed, kind):
    snap = variant(n, seed, kind)
    assert_same(device_step(snap.copy(), sort_path=SORT_PATH.get(kind)), run_step(snap.copy()))


@pytest.mark.parametrize("flags", [dict(enable_coordinator=False), dict(enable_coscheduler=False)])
def test_ablations_match_oracle(flags):
    snap = snapshot_v1(40_000, seed=31, pool="pressure")
    assert_same(device_step(snap.copy(), **flags), run_step(snap.copy(), **flags))


def test_step_without_control_matches_oracle():
    snap = snapshot_v1(50_000, seed=32, pool="pressure")
    assert_same(device_step(snap.copy(), control_due=False),
                run_step(snap.copy(), control_due=False))


def test_one_million_sessions_match_oracle():
    snap = snapshot_v1(1_000_000, seed=0, pool="headroom")
    assert_same(device_step(snap.copy()), run_step(snap.copy()))


def test_restore_replays_identically():
    snap = snapshot_v1(60_000, seed=41, pool="pressure")
    eng = MarsEngine(max_rows=snap.n, max_queue=len(snap.queue),
                     config=make_config(initial_window=snap.initial_window))
    eng.load_snapshot(snap)
    eng.checkpoint()
    si = eng.step_in(snap.now, True, snap.active_tools, 0, snap.worker_slots)
    a = canon(canonical(eng.step(si), eng, snap))
    eng.restore()
    b = canon(canonical(eng.step(si), eng, snap))
    eng.set_graph(True)  # whole-step CUDA graph replays the same decisions
    for _ in range(2):
        eng.restore()
        c = canon(canonical(eng.step(si), eng, snap))
        assert c == a
    eng.close()
    assert a == b


def test_retention_batch_matches_reference_kat():
    kat = json.load(open(os.path.join(GOLDEN, "kat.json")))["retention"]
    eng = MarsEngine(max_rows=16, max_queue=1)
    for r in kat:
        ema = r["ema"] if r["ema"] is not None else 5.0
        pin, b, c, d = eng.retention_batch(np.array([r["ctx"]]), np.array([r["kv"]]), r["total"],
                                           r["usage"], ema, r["now"])
        assert (bool(pin[0]), float(b[0]), float(c[0]), float(d[0])) == (
            r["pin"], r["benefit"], r["cost"], r["deadline"])
    eng.close()


@pytest.mark.parametrize("policy", ["fcfs", "program_priority", "static_ttl", "dynamic_ttl"])
@pytest.mark.parametrize("pool,n,seed", [("headroom", 100_000, 51), ("pressure", 20_000, 52)])
def test_comparison_policy_step_matches_oracle(policy, pool, n, seed):
    """The reference's comparison policies (baselines.py:108-315) on the same
    device step: window order, whole-chunk fitting, head-of-line blocking,
    their reclaim orders (exact full-table search) and the TTL pin rule."""
    snap = comparison_variant(n, seed, policy, pool)
    got = device_step(snap.copy(), control_due=False, policy=policy)
    want = run_step(snap.copy(), control_due=False, policy=policy)
    assert_same(got, want)
    if pool == "pressure":
        assert want["evictions"], "the pressure case must exercise the reclaimer"


def test_unstaged_emission_matches_oracle(monkeypatch):
    """A CTA whose emitted entries exceed k_scan's staging area writes its
    row lists straight to the global lists and gathers from there (forced
    here with MARS_SCAN_NO_STAGE=1; read at context creation)."""
    monkeypatch.setenv("MARS_SCAN_NO_STAGE", "1")
    for kind, n, seed in (("headroom", 200_000, 61), ("expired_big", 150_000, 62)):
        snap = variant(n, seed, kind)
        assert_same(device_step(snap.copy()), run_step(snap.copy()))


@pytest.mark.parametrize("kind", ["queue_shuffled", "desc_sorted"])
def test_pack_sort_inside_control_plane_matches_oracle(kind, monkeypatch):
    """The big-list sort inside k_control (MARS_PACK_CTAS=0: no early k_pack)."""
    monkeypatch.setenv("MARS_PACK_CTAS", "0")
    snap = variant(60_000, 71, kind)
    assert_same(device_step(snap.copy(), sort_path=1), run_step(snap.copy()))


@pytest.mark.parametrize("n", [1, 2, 3, 17, 129, 2049, 4097])
@pytest.mark.parametrize("pool", ["headroom", "pressure"])
def test_tiny_tables_match_oracle(n, pool):
    """Edge sizes: fewer rows than the window, one TMA round, a partial last
    round, the small-queue pack, one row per CTA."""
    snap = snapshot_v1(n, seed=1000 + n, pool=pool)
    assert_same(device_step(snap.copy()), run_step(snap.copy()))


@pytest.mark.parametrize("policy", ["fcfs", "program_priority", "static_ttl"])
@pytest.mark.parametrize("n", [3, 129, 4097])
def test_tiny_tables_comparison_policies_match_oracle(policy, n):
    snap = comparison_variant(n, 2000 + n, policy, "pressure")
    assert_same(device_step(snap.copy(), control_due=False, policy=policy),
                run_step(snap.copy(), control_due=False, policy=policy))


def test_no_ready_rows_matches_oracle():
    """Every session waits for admission or sits in a tool call: no window."""
    from paper_2604_26963_b200.snapshot import DECODE, PREFILL, TOOL

    snap = snapshot_v1(5000, seed=77, pool="headroom")
    c = snap.cols
    ready = (c["phase"] == DECODE) | (c["phase"] == PREFILL)
    held = (-(-c["kv"][ready].astype(np.int64) // 16)).sum()
    c["phase"][ready] = TOOL
    c["kv"][ready] = 0
    c["flags"][ready] &= ~np.uint8(8)  # no boundary rows left
    snap.free_blocks += int(held)
    assert_same(device_step(snap.copy()), run_step(snap.copy()))


def test_pack_sort_inside_control_plane_multi_batch(monkeypatch):
    """The in-control LSD with ~4K list entries per CTA (the sharded union
    list's regime): several 1024-entry scatter batches per CTA and pass."""
    monkeypatch.setenv("MARS_PACK_CTAS", "0")
    monkeypatch.setenv("MARS_CTL_PER_CTA", "4096")
    for kind in ("queue_shuffled", "desc_sorted", "hot_req"):
        snap = variant(200_000, 72, kind)
        assert_same(device_step(snap.copy(), sort_path=1), run_step(snap.copy()))


@pytest.mark.parametrize("pool", ["headroom", "pressure"])
def test_step_reads_only_its_columns(pool):
    """engine.step_columns (the e2e upload set): the columns it leaves out
    cannot change the step's decisions in that configuration."""
    from paper_2604_26963_b200.engine import step_columns
    snap = snapshot_v1(60_000, seed=7, pool=pool)
    want = device_step(snap.copy())
    junk = snap.copy()
    rng = np.random.default_rng(3)
    keep = set(step_columns())
    for k, a in junk.cols.items():
        if k in keep:
            continue
        if a.dtype.kind == "f":
            junk.cols[k] = rng.uniform(-1e6, 1e6, a.shape).astype(a.dtype)
        else:
            junk.cols[k] = rng.integers(0, 1000, a.shape).astype(a.dtype)
    assert keep != set(snap.cols)
    got = device_step(junk)
    for k in got["state"]:   # the end-state dump shows the junk itself
        if k not in keep:
            got["state"][k] = want["state"][k]
    assert canon(got) == canon(want)


@pytest.mark.parametrize("pool", ["headroom", "pressure"])
def test_fast_fetch_matches_field_by_field(pool):
    """engine.fetch (one gather launch into the pinned arena, arrays sliced
    from one view of it) against the field-by-field conversion."""
    from dataclasses import fields
    snap = snapshot_v1(60_000, seed=11, pool=pool)
    eng = MarsEngine(max_rows=snap.n, max_queue=len(snap.queue),
                     config=make_config(initial_window=snap.initial_window))
    eng.load_snapshot(snap)
    si = eng.step_in(snap.now, True, snap.active_tools, snap.queued_tools, snap.worker_slots)
    a = eng.step(si)
    b = eng.fetch_reference()
    for f in fields(a):
        x, y = getattr(a, f.name), getattr(b, f.name)
        if isinstance(x, np.ndarray):
            assert x.dtype == y.dtype and np.array_equal(x, y), f.name
        else:
            assert x == y, f.name
    assert len(a.ret_rows) > 0 and len(a.journal_op) > 0
    assert pool == "pressure" or len(a.admitted_rows) > 0
    eng.close()


@pytest.mark.parametrize("extra", [0, 5000])
def test_input_arena_upload_then_step_matches_oracle(extra):
    """mars_input_arena + mars_upsert_arena (the bench's e2e upload): the
    step columns written into the pinned arena, the device table clobbered,
    then rows [0, n) uploaded -- one linear copy of the whole table when n is
    the capacity (extra 0), one pitched copy per element-size group
    otherwise; the step sees every byte.  n < max_rows: the copies stop at
    row n."""
    from paper_2604_26963_b200.engine import step_columns

    snap = snapshot_v1(150_000, seed=43, pool="pressure")
    eng = MarsEngine(max_rows=snap.n + extra, max_queue=len(snap.queue),
                     config=make_config(initial_window=snap.initial_window))
    eng.load_snapshot(snap)
    names = step_columns()
    arena = eng.input_arena()
    for k in names:
        arena[k][:snap.n] = snap.cols[k]
        arena[k][snap.n:] = 0
    tail = np.arange(snap.n, snap.n + extra)
    before = eng.read(["phase"], rows=tail)["phase"] if extra else None
    eng.upsert({k: np.zeros_like(snap.cols[k]) for k in names})  # clobbered ...
    eng.upsert_arena(snap.n, names)                              # ... restored
    if extra:
        assert np.array_equal(before, eng.read(["phase"], rows=tail)["phase"])  # past n untouched
    si = eng.step_in(snap.now, True, snap.active_tools, snap.queued_tools, snap.worker_slots)
    res = eng.step(si)
    got = canonical(res, eng, snap, True)
    eng.close()
    assert res.status == 0, res.status
    assert_same(got, run_step(snap.copy()))
