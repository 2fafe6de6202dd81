"""Consecutive device ticks (MARS_MODE_ADVANCE): the
tick's tail -- step_gpu on the plan and the rounds that end (note_round_blocks,
DONE on the last round, pin or free at the tool boundary) -- runs on the
device, so the session table evolves across steps without a host round trip.
Every tick's decisions and the end-of-run table, pins and scalars must equal
the CPU oracle's multi-tick restatement (oracle/snapshot_step.py:run_ticks)."""

import numpy as np
import pytest

from oracle.snapshot_step import run_ticks
from paper_2604_26963_b200 import _native as N
from paper_2604_26963_b200.engine import MarsEngine, canonical, make_config
from paper_2604_26963_b200.snapshot import F_PINNED, snapshot_v1
from tests._canon import canon

pytestmark = pytest.mark.gpu


def device_ticks(snap, ticks, control_ticks=(0,), resumes=None, **flags):
    eng = MarsEngine(max_rows=snap.n, max_queue=max(len(snap.queue), 1),
                     config=make_config(**flags, initial_window=snap.initial_window))
    eng.load_snapshot(snap)
    tick = eng.cfg.tick_duration_s
    now = snap.now
    outs, diags = [], []
    for k in range(ticks):
        due = k in control_ticks
        if resumes and k in resumes:
            r, fin, dur, newp, dec = map(list, zip(*resumes[k]))
            diags.append(eng.resume(r, fin, dur, newp, dec, now))
        si = eng.step_in(now, due, snap.active_tools, snap.queued_tools, snap.worker_slots,
                         N.MODE_ADVANCE)
        res = eng.step(si)
        assert res.status == 0, res.status
        out = canonical(res, eng, snap, due)
        if k < ticks - 1:
            out.pop("state")
        outs.append(out)
        diags.append(res.diag)
        now = now + tick
    pins = eng.read(["flags", "deadline", "pinned_blocks", "plevel"])
    sc = eng.get_scalars()
    eng.close()
    return outs, diags, pins, sc


@pytest.mark.parametrize("n,seed,pool,ticks", [(20_000, 81, "headroom", 8),
                                               (20_000, 82, "pressure", 8),
                                               (200_000, 83, "headroom", 4)])
def test_device_ticks_match_oracle(n, seed, pool, ticks):
    snap = snapshot_v1(n, seed=seed, pool=pool)
    got, diags, pins, sc = device_ticks(snap.copy(), ticks)
    want, w = run_ticks(snap.copy(), ticks)
    for k in range(ticks):
        g, o = canon(got[k]), canon(want[k])
        for key in o:
            assert g[key] == o[key], f"tick {k}: {key} differs"
    assert sum(d["n_round_end"] for d in diags if "n_round_end" in d) > 0, \
        "no round ended: the tail was not exercised"
    # pins taken at tool boundaries (PinnedSession, baselines.py:386-394)
    pinned = (pins["flags"] & F_PINNED) != 0
    rows = {w.row_of[sid]: ps for sid, ps in w.policy.pinned.items()}
    assert set(np.nonzero(pinned)[0].tolist()) == set(rows)
    for r, ps in rows.items():
        assert pins["deadline"][r] == ps.retention_deadline
        assert pins["pinned_blocks"][r] == ps.pinned_blocks
        assert pins["plevel"][r] == ps.level
    # pool and telemetry after the tail
    assert sc.free_blocks == w.pool.free_blocks
    assert (sc.ema_blocks if sc.has_ema_blocks else None) == w.tel.ema_blocks_per_session


@pytest.mark.parametrize("policy", ["fcfs", "static_ttl"])
def test_device_ticks_comparison_policies_match_oracle(policy):
    from tests._variants import comparison_variant

    snap = comparison_variant(20_000, 84, policy, "pressure")
    got, _, _, sc = device_ticks(snap.copy(), 6, control_ticks=(), policy=policy)
    want, w = run_ticks(snap.copy(), 6, control_ticks=(), policy=policy)
    for k in range(6):
        g, o = canon(got[k]), canon(want[k])
        for key in o:
            assert g[key] == o[key], f"tick {k}: {key} differs"
    assert sc.free_blocks == w.pool.free_blocks


def test_device_ticks_with_tool_returns_match_oracle():
    """resume_from_tool on the device (mars_resume, sim.py:190-231): warm
    resumes (the pin covers the finish time), cold ones, pins that expired
    before the return, then the resumed rounds run through the next ticks."""
    from oracle.core import TOOL

    snap = snapshot_v1(20_000, seed=85, pool="headroom")
    _, w0 = run_ticks(snap.copy(), 2)
    tool_rows = [r for r, s in enumerate(w0.sessions)
                 if s.phase == TOOL and not s.is_last_round][:400]
    # pins that survive the expiry of ticks 0-1 but not the tool's finish at
    # tick 2 (evicted at return, sim.py:210-214)
    late = [r for r in tool_rows if snap.cols["flags"][r] & F_PINNED][:40]
    snap.cols["deadline"][late] = snap.now + 0.1
    now2 = snap.now + w0.gpu.tick_duration_s + w0.gpu.tick_duration_s
    plan = [(r, now2 if r in late else now2 - (i % 7) * 5.0, 1.0 + (i % 11) * 0.5,
             32 + r % 200, 2 + r % 9) for i, r in enumerate(tool_rows)]
    resumes = {2: plan}
    got, diags, pins, sc = device_ticks(snap.copy(), 6, resumes=resumes)
    want, w = run_ticks(snap.copy(), 6, resumes=resumes)
    for k in range(6):
        g, o = canon(got[k]), canon(want[k])
        for key in o:
            assert g[key] == o[key], f"tick {k}: {key} differs"
    counts = [d for d in diags if "warm" in d][0]
    assert counts["warm"] > 0 and counts["cold"] > 0 and counts["evicted"] > 0, counts
    assert sc.free_blocks == w.pool.free_blocks
    assert sc.ema_tool == w.tel.ema_tool_duration
    pinned = (pins["flags"] & F_PINNED) != 0
    assert set(np.nonzero(pinned)[0].tolist()) == {w.row_of[sid] for sid in w.policy.pinned}
