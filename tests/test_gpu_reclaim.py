"""Heavy reclamation and tick-gridded ties on the device (through the C ABI).

* every policy's reclaimer taking dozens of one- and two-block victims in one
  step (scheduler.py:228-267, baselines.py:118-140, 176-186, 264-298), with
  and without exact time ties on the tick grid: against steps frozen from the
  reference itself (30K sessions, tests/golden/heavy_steps.json) and from the
  oracle at 1M sessions (tests/golden/heavy_1m.json);
* the victim stream k_scan selects covers every claim: the walk never falls
  back to its exact full-table search on these tables;
* the grid radix refinement of the candidate lists (forced with low
  triggers) and the full-table fallback (forced with a 4-entry stream) still
  reproduce the oracle.
"""

import json
import os

import pytest

from oracle.make_golden import heavy_kw, heavy_snapshot
from oracle.snapshot_step import run_step
from paper_2604_26963_b200.engine import MarsEngine, canonical, make_config
from paper_2604_26963_b200.snapshot import snapshot_v1
from tests._canon import canon, digest
from tests._variants import comparison_variant, reclaim_heavy, tick_grid, variant
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

HEAVY = json.load(open(os.path.join(GOLDEN, "heavy_steps.json")))
HEAVY_1M = json.load(open(os.path.join(GOLDEN, "heavy_1m.json")))


def device_step(snap, control_due=True, **flags):
    eng = MarsEngine(max_rows=snap.n, max_queue=max(len(snap.queue), 1),
                     config=make_config(**flags, initial_window=snap.initial_window))
    eng.load_snapshot(snap)
    si = eng.step_in(snap.now, control_due, snap.active_tools, snap.queued_tools,
                     snap.worker_slots)
    res = eng.step(si)
    out = canonical(res, eng, snap, control_due)
    eng.close()
    assert res.status == 0, res.status
    return out, res.diag


def assert_same(got, want):
    g, w = canon(got), canon(want)
    for k in w:
        if g[k] != w[k]:
            gs, ws = json.dumps(g[k]), json.dumps(w[k])
            raise AssertionError(f"{k} differs:\n device {gs[:600]}\n oracle {ws[:600]}")


def _flags(case):
    kw = heavy_kw(case)
    return kw.pop("control_due"), kw


@pytest.mark.parametrize("i", range(len(HEAVY)))
def test_heavy_step_matches_reference_golden(i):
    case = HEAVY[i]["case"]
    due, kw = _flags(case)
    got, diag = device_step(heavy_snapshot(case), control_due=due, **kw)
    got = canon(got)
    for k, v in HEAVY[i]["out"].items():
        assert got[k] == v, k
    if case["kind"] == "reclaim_heavy":
        assert len(got["evictions"]) >= 40
    assert diag["n_fullscan"] == 0, diag


@pytest.mark.parametrize("i", range(len(HEAVY_1M)))
def test_heavy_step_1m_matches_oracle_golden(i):
    case = HEAVY_1M[i]["case"]
    due, kw = _flags(case)
    got, diag = device_step(heavy_snapshot(case), control_due=due, **kw)
    got = digest(canon(got))
    for k, v in HEAVY_1M[i]["out"].items():
        assert got[k] == v, k
    assert diag["n_fullscan"] == 0, diag
    # one- and two-block victims tie on (level, blocks) across ~100K rows:
    # where the digits cannot cut the victim list, the grid refinement does
    assert (diag["ref_flags"] & 2) or diag["n_victim_cand"] <= 1024, diag
    if case["policy"] == "mars" and case.get("enable_coordinator", True):
        assert diag["ref_flags"] & 2, diag


@pytest.mark.parametrize("policy", ["mars", "program_priority"])
def test_heavy_step_100k_matches_oracle(policy):
    snap = tick_grid(reclaim_heavy(100_000, 101, policy), 101)
    due = policy == "mars"
    got, diag = device_step(snap.copy(), control_due=due, policy=policy)
    assert_same(got, run_step(snap.copy(), control_due=due, policy=policy))
    assert diag["n_fullscan"] == 0


@pytest.mark.parametrize("pool", ["headroom", "pressure"])
def test_tick_grid_1m_matches_oracle(pool):
    """Ready times, wait times and arrivals on the tick grid with a batch
    admitted at `now`: exact ties in the window key, decided by session id."""
    snap = tick_grid(snapshot_v1(1_000_000, seed=111, pool=pool), 111)
    got, _ = device_step(snap.copy())
    assert_same(got, run_step(snap.copy()))


@pytest.mark.parametrize("kind,policy", [("reclaim_heavy", "mars"), ("reclaim_heavy", "fcfs"),
                                         ("tick_grid", "mars"), ("headroom", "mars"),
                                         ("pressure", "static_ttl")])
def test_forced_refinement_matches_oracle(kind, policy, monkeypatch):
    """Refine both candidate lists whatever their length (triggers at their
    targets): the grid radix select and the admission's refined-list append."""
    monkeypatch.setenv("MARS_REF_TRIG_W", "1")
    monkeypatch.setenv("MARS_REF_TRIG_V", "1")
    if kind == "reclaim_heavy":
        snap = tick_grid(reclaim_heavy(60_000, 121, policy), 121)
    elif kind == "tick_grid":
        snap = tick_grid(snapshot_v1(60_000, seed=122, pool="headroom"), 122)
    elif policy == "mars":
        snap = variant(60_000, 123, kind)
    else:
        snap = comparison_variant(60_000, 124, policy, kind)
    due = policy == "mars"
    got, diag = device_step(snap.copy(), control_due=due, policy=policy)
    assert_same(got, run_step(snap.copy(), control_due=due, policy=policy))
    assert (diag["ref_flags"] & 1) or diag["n_window_cand"] <= 128, diag
    assert (diag["ref_flags"] & 2) or diag["n_victim_cand"] <= 512, diag


@pytest.mark.parametrize("policy", ["mars", "fcfs", "program_priority", "dynamic_ttl"])
def test_full_table_fallback_matches_oracle(policy, monkeypatch):
    """A 4-entry victim stream: claims exhaust it and take the walk's exact
    full-table reclaimer."""
    monkeypatch.setenv("MARS_VSTREAM", "4")
    snap = reclaim_heavy(20_000, 131, policy)
    due = policy == "mars"
    got, diag = device_step(snap.copy(), control_due=due, policy=policy)
    assert_same(got, run_step(snap.copy(), control_due=due, policy=policy))
    assert diag["n_fullscan"] > 0, diag
