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


def device_ticks(snap, ticks, control_ticks=(0,), **flags):
    eng = MarsEngine(max_rows=snap.n, max_queue=max(len(snap.queue), 1),
                     config=make_config(**flags, initial_window=snap.initial_window))
    eng.load_snapshot(snap)
    tick = eng.cfg.tick_duration_s
    now = snap.now
    outs, diags = [], []
    for k in range(ticks):
        due = k in control_ticks
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
    assert sum(d["n_round_end"] for d in diags) > 0, "no round ended: the tail was not exercised"
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
