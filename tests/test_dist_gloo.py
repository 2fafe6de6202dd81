"""World-size-2 test of the sharded engine's exchange protocol on CPU (gloo).

Each rank encodes its replica's probe counters and admission list in the
wire format of the device kernels (k_export_queue), runs the same
collectives the GPU path runs (``paper_2604_26963_b200.dist.exchange``), and
decodes the union list exactly as k_build_global_queue does; the global
admission over it must equal the sharded oracle (oracle/multi.py) on both
ranks.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import admission as oa
from oracle import core as oc
from oracle.multi import run_multi_step
from oracle.snapshot_step import ToolCounts, World
from paper_2604_26963_b200.dist import (COUNTERS, XQ_NONE, decode_gathered, encode_queue, exchange,
                                        interleaved_gpos)
from paper_2604_26963_b200.snapshot import snapshot_shard, snapshot_v1

N_PER_RANK = 1500
WORLD = 2


def shards(kind="independent"):
    if kind == "global":
        # config (3): ONE global snapshot, rows sharded rank mod G, every
        # admission entry at its position in the global list
        glob = snapshot_v1(WORLD * N_PER_RANK, seed=95, pool="headroom")
        snaps = [snapshot_shard(glob, WORLD, g, box_global=True) for g in range(WORLD)]
        return snaps, [s.meta["gpos"].tolist() for s in snaps]
    snaps = [snapshot_v1(N_PER_RANK, seed=90 + g, pool="headroom") for g in range(WORLD)]
    gpos = interleaved_gpos([len(s.queue) for s in snaps])
    return snaps, gpos


def _worker(rank, port, out, kind="independent"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    snaps, gpos = shards(kind)
    snap = snaps[rank]
    w = World(snap)
    # replica-local expiry + probe (what k_scan leaves in xc)
    for sid in w.policy.expired_pins(snap.now):
        w.pool.release_pinned(sid)
        w.policy.on_evicted(sid)
    w.tel.probe(w.pool, ToolCounts(snap.active_tools, snap.queued_tools), len(w.active))
    xc = torch.tensor([w.tel.available_kv, w.pool.total_blocks, w.tel.active_sessions,
                       len(w.queue), 0, 0, 0, 0], dtype=torch.int64)
    q = snap.queue
    cap = 2048
    send = torch.from_numpy(encode_queue(gpos[rank], snap.cols["req_blocks"][q],
                                         (snap.cols["flags"][q] & 16) != 0, cap).view(np.int64))
    recv = torch.zeros(WORLD * send.numel(), dtype=torch.int64)
    exchange(xc[:len(COUNTERS)], send, recv, None)
    req, lng, owner, row = decode_gathered(recv.numpy().view(np.uint64), WORLD, cap, rank, q)
    # global admission over the union list with pooled telemetry
    avail, total, active = int(xc[0]), int(xc[1]), int(xc[2])
    T = oa.Counters(total)
    T.available_kv = avail
    T.kv_usage_ratio = (total - avail) / total
    T.active_sessions = active
    T.active_tools, T.queued_tools = snap.active_tools, snap.queued_tools
    T.ema_tool_duration = snap.ema_tool
    oa.refresh_pressure(T, oa.Pressure(), snap.worker_slots)
    entries = [oa.Pending(oc.Session(f"q{i:07d}", [oc.Round(1, 1)], 0.0), int(r), bool(l), 0.0)
               for i, (r, l) in enumerate(zip(req, lng))]
    pos = {id(e): i for i, e in enumerate(entries)}
    ctl = oa.Controller(initial_window=snap.initial_window)
    adm = oa.admit_step(entries, ctl, T, snap.worker_slots, oa.Pressure(), snap.now)
    got = [(int(owner[pos[id(e)]]), int(row[pos[id(e)]])) for e in adm]
    out[rank] = (got, int(xc[3]), ctl.w_adm)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("kind", ["independent", "global"])
def test_two_rank_exchange_reproduces_the_sharded_oracle(kind):
    snaps, gpos = shards(kind)
    want = run_multi_step([s.copy() for s in snaps], gpos)["control"]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(_free_port(), out, kind), nprocs=WORLD, join=True)
    for rank in range(WORLD):
        got, qlen, w_adm = out[rank]
        # the same winners in the same order on every rank; a rank knows the
        # rows of its own entries only (the wire carries no rows)
        assert got == [(o, r if o == rank else XQ_NONE) for o, r in want["admitted_global"]]
        assert qlen == sum(len(s.queue) for s in snaps)
        assert w_adm == want["w_adm"]
