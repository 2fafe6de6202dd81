"""Sharded engine on the device.

* world 1: the phase-split step with the exchange must reproduce the
  single-replica step exactly;
* world 2 on ONE GPU: two replica contexts, the all-reduce / all-gather done
  by hand on the device buffers (what NCCL does across GPUs), against the
  sharded oracle (oracle/multi.py).
"""

import numpy as np
import pytest
import torch

from oracle.multi import run_multi_step
from paper_2604_26963_b200.dist import COUNTERS, ShardedEngine, interleaved_gpos
from paper_2604_26963_b200.engine import MarsEngine, canonical, make_config
from paper_2604_26963_b200.snapshot import F_LONG, snapshot_shard, snapshot_v1
from tests._canon import canon

pytestmark = pytest.mark.gpu


def _replica(snap, world, rank, gpos, cap=None):
    # every replica exchanges the same fixed-size buffers: one capacity for all
    cap = cap or max(len(snap.queue), 1) * 2
    eng = MarsEngine(max_rows=snap.n, max_queue=cap,
                     config=make_config(initial_window=snap.initial_window))
    eng.load_snapshot(snap)
    sh = ShardedEngine(eng, world=world, rank=rank)
    q = snap.queue
    sh.set_queue(q, snap.cols["req_blocks"][q], (snap.cols["flags"][q] & F_LONG) != 0, gpos)
    return eng, sh


@pytest.mark.parametrize("pool", ["headroom", "pressure"])
def test_world_one_sharded_step_equals_the_single_step(pool):
    snap = snapshot_v1(40_000, seed=61, pool=pool)
    eng = MarsEngine(max_rows=snap.n, max_queue=len(snap.queue),
                     config=make_config(initial_window=snap.initial_window))
    eng.load_snapshot(snap)
    si = eng.step_in(snap.now, True, snap.active_tools, 0, snap.worker_slots)
    want = canon(canonical(eng.step(si), eng, snap))
    eng.close()
    eng2, sh = _replica(snap, 1, 0, np.arange(len(snap.queue)))
    res = sh.step(eng2.step_in(snap.now, True, snap.active_tools, 0, snap.worker_slots))
    assert res.status == 0
    got = canonical(res, eng2, snap)
    rows, gpos = sh.get_queue()
    got["control"]["queue"] = [int(r) for r in rows[np.argsort(gpos, kind="stable")]]
    got = canon(got)
    for k in want:
        assert got[k] == want[k], k
    eng2.close()


@pytest.mark.parametrize("kind,world", [("independent", 2), ("global", 2), ("global", 4)])
def test_replicas_on_one_gpu_match_the_sharded_oracle(kind, world):
    """Replica contexts on one GPU, the collectives done by hand.  "global":
    config (3) -- ONE snapshot_v1 sharded rank mod G with box-global tool
    counters, every admission entry at its global list position."""
    if kind == "global":
        glob = snapshot_v1(30_000 * world, seed=77, pool="headroom")
        # a window that admits part of the union list: the residual's global
        # order (packed order, dense positions) is exercised
        glob.initial_window = 2000.0
        glob.worker_slots = 4000
        snaps = [snapshot_shard(glob, world, g, box_global=True) for g in range(world)]
        gpos = [s.meta["gpos"] for s in snaps]
    else:
        snaps = [snapshot_v1(30_000, seed=70 + g, pool="headroom") for g in range(world)]
        gpos = interleaved_gpos([len(s.queue) for s in snaps])
    want = run_multi_step([s.copy() for s in snaps], gpos)
    cap = 2 * max(len(s.queue) for s in snaps)
    reps = [_replica(s, world, g, gpos[g], cap) for g, s in enumerate(snaps)]
    sis = [e.step_in(s.now, True, s.active_tools, 0, s.worker_slots) for (e, _), s in
           zip(reps, snaps)]
    for (e, sh), si in zip(reps, sis):
        sh.phase(si, 1)
        e._check(e.lib.mars_sync(e.ctx))
    # the collectives, by hand: sum of counters, rank-major concatenation
    xc = sum(sh.xc[:len(COUNTERS)].clone() for _, sh in reps)
    recv = torch.cat([sh.xsend.clone() for _, sh in reps])
    for e, sh in reps:
        sh.xc[:len(COUNTERS)].copy_(xc)
        sh.xrecv.copy_(recv)
        torch.cuda.synchronize()
    for g, ((e, sh), si, s) in enumerate(zip(reps, sis, snaps)):
        sh.phase(si, 2)
        res = e.fetch()
        assert res.status == 0
        got = canonical(res, e, s)
        mine = want["replicas"][g]
        assert got["window"] == mine["window"]
        assert got["decodes"] == mine["decodes"]
        assert got["prefills"] == mine["prefills"]
        assert got["evictions"] == mine["evictions"]
        assert got["expired"] == mine["expired"]
        assert got["control"]["admitted"] == want["control"]["admitted"][g]
        rows, gp = sh.get_queue()
        order = np.argsort(gp, kind="stable")
        assert [(int(r), int(p)) for r, p in zip(rows[order], gp[order])] == \
            [tuple(x) for x in want["control"]["residual"][g]]
        assert canon(got)["retention"] == canon({"r": mine["retention"]})["r"]
        for k in mine["state"]:
            assert np.array_equal(got["state"][k], mine["state"][k]), k
        e.close()


def test_sharded_step_as_one_cuda_graph_replays_the_eager_step():
    """phase 1 + the exchange + phase 2 captured as ONE CUDA graph
    (ShardedEngine.capture; the bench's multi-GPU step) and replayed from a
    restored state give the eager sharded step's outputs (world 1: the
    exchange is the device copy the collectives reduce to)."""
    snap = snapshot_v1(30_000, seed=81, pool="headroom")
    eng, sh = _replica(snap, 1, 0, np.arange(len(snap.queue)))
    si = eng.step_in(snap.now, True, snap.active_tools, 0, snap.worker_slots)
    eng.checkpoint()
    want = canon(canonical(sh.step(si), eng, snap))
    eng.restore()
    sh.capture(si)
    for _ in range(2):
        eng.restore()
        sh.replay()
        got = canon(canonical(eng.fetch(), eng, snap))
        for k in want:
            assert got[k] == want[k], k
    eng.close()
