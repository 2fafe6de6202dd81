"""Oracle for the sharded (multi-GPU) scheduling step.

The reference has no multi-replica semantics (multi-GPU is future work,
PAPER.md:549-550).  The B200 build shards sessions across GPUs as
data-parallel engine replicas; this module is the written-down semantics
the device path must reproduce, composed only of reference functions:

* every replica g owns its own session rows, KV pool, token budget and
  window; pin expiry, the probe, S2 retention and S4 planning are
  replica-local (the single-GPU step on that replica);
* the control plane is global: pooled telemetry -- available_kv = sum(free_g),
  total = sum(total_g), kv_usage_ratio = (total - sum(free_g)) / total,
  active_sessions = sum(active_g) (tool counters are box-global) -- feeds one
  refresh_pressure and ONE balance_and_admit over the union admission list
  in global list order (``gpos``); each replica then admits its own
  entries, and the residual keeps global packed order (dense new gpos).

With one replica this is exactly ``snapshot_step.run_step``.  TEST
INFRASTRUCTURE ONLY.
"""

from __future__ import annotations

from typing import Dict, List, Optional, Sequence

from . import admission as adm
from .core import PREFILL, DECODE, submit_round
from .policy import retention
from .snapshot_step import ToolCounts, World, extract_state


def pooled_probe(worlds: Sequence[World], active_tools: int, queued_tools: int) -> adm.Counters:
    total = sum(w.pool.total_blocks for w in worlds)
    free = sum(w.pool.free_blocks for w in worlds)
    t = adm.Counters(total)
    t.available_kv = free
    t.kv_usage_ratio = (total - free) / total
    t.active_sessions = sum(len(w.active) for w in worlds)
    t.active_tools = active_tools
    t.queued_tools = queued_tools
    return t


def run_multi_step(snaps: Sequence, gpos: Sequence[Sequence[int]], control_due: bool = True,
                   telemetry_state: Optional[dict] = None, **kw) -> dict:
    """One sharded step.  ``gpos[g][k]`` is the global list position of the k-th
    entry of replica g's queue (positions are a permutation of 0..Q-1)."""
    worlds = [World(s, **kw) for s in snaps]
    s0 = snaps[0]
    now = s0.now
    per = []
    # 1. replica-local expiry + probe
    for w, s in zip(worlds, snaps):
        expired = []
        for sid in w.policy.expired_pins(now):
            expired.append((w.row_of[sid], _evict_pinned(w, sid)))
        w.tel.probe(w.pool, ToolCounts(s.active_tools, s.queued_tools), len(w.active))
        per.append({"expired": expired})
    # 2. pooled telemetry, replicated controller
    T = pooled_probe(worlds, s0.active_tools, s0.queued_tools)
    T.ema_tool_duration = s0.ema_tool
    T.ema_blocks_per_session = s0.ema_blocks
    T.blocks_seed = s0.blocks_seed
    for k, v in (telemetry_state or {}).items():
        setattr(T, k, v)
    ctl = adm.Controller(initial_window=s0.initial_window)
    control = None
    if control_due:
        adm.refresh_pressure(T, worlds[0].pressure, s0.worker_slots)
        gq = []
        for g, w in enumerate(worlds):
            for k, e in enumerate(w.queue):
                gq.append((gpos[g][k], g, e))
        gq.sort(key=lambda x: x[0])
        owner = {id(e): g for _, g, e in gq}
        queue = [e for _, _, e in gq]
        stats: dict = {}
        admitted = adm.admit_step(queue, ctl, T, s0.worker_slots, worlds[0].pressure, now, None,
                                  stats)
        adm_rows: List[List[int]] = [[] for _ in worlds]
        for e in admitted:
            g = owner[id(e)]
            w = worlds[g]
            s = e.call
            s.admit_time = now
            submit_round(s, now)
            T.record("gpu_submit", {"projected_blocks": s.incremental_blocks(
                s.remaining_prefill, w.pool.block_size)})
            w.active[s.session_id] = s
            w.policy.on_admit(s, now)
            adm_rows[g].append(w.row_of[s.session_id])
        res_rows: List[List[tuple]] = [[] for _ in worlds]
        for j, e in enumerate(queue):
            g = owner[id(e)]
            res_rows[g].append((worlds[g].row_of[e.call.session_id], j))
        for g, w in enumerate(worlds):
            mine = set(r for r, _ in res_rows[g])
            w.queue = [e for e in w.queue if w.row_of[e.call.session_id] in mine]
        control = dict(w_adm=ctl.w_adm, last_update=ctl.last_update, limit=stats["limit"],
                       slots=stats["slots"], take=stats["take"],
                       cpu_overloaded=T.cpu_overloaded, kv_overloaded=T.kv_overloaded,
                       blocks_seed=T.blocks_seed, available_kv=T.available_kv,
                       admitted=adm_rows, residual=res_rows,
                       admitted_global=[(owner[id(e)], worlds[owner[id(e)]].row_of[
                           e.call.session_id]) for e in admitted])
    # 3. replica-local S2 + S4 on the local pool and local probe
    for g, (w, s) in enumerate(zip(worlds, snaps)):
        pol, pool, tel = w.policy, w.pool, w.tel
        ret = []
        for r in w.boundary:
            d = retention(w.sessions[r], tel, pool, w.gpu, pol.retention, w.pressure, now)
            ret.append((r, d.pin, d.benefit_s, d.cost_s, d.retention_deadline))
        ready = sorted((x for x in w.active.values() if x.phase in (PREFILL, DECODE)),
                       key=lambda x: x.session_id)
        row = w.row_of

        def plan_evict(v, w=w):
            _evict(w, v.session_id, v.kind)

        plan = pol.plan_tick(ready, pool, w.gpu, tel, now, plan_evict) if ready else None
        per[g].update(
            retention=ret, window=[row[x.session_id] for x in pol.last_window],
            decodes=[row[x] for x in plan.decode_ids] if plan else [],
            prefills=[(row[x], gr) for x, gr in plan.prefill_grants] if plan else [],
            evictions=[(row[v.session_id], v.kind, v.blocks) for v in plan.evictions]
            if plan else [],
            total_tokens=plan.total_tokens if plan else 0, free_blocks=pool.free_blocks,
            state=extract_state(w))
    return {"replicas": per, "control": control,
            "pooled": dict(available_kv=sum(w.pool.free_blocks for w in worlds))}


def _evict_pinned(w: World, sid: str) -> int:
    return _evict(w, sid, "pinned")


def _evict(w: World, sid: str, kind: str) -> int:
    s = w.policy.calls[sid]
    if kind == "pinned":
        n = w.pool.release_pinned(sid)
        s.pinned = False
        s.retention_deadline = None
    else:
        n = w.pool.free(sid)
    s.kv_tokens = 0
    if kind == "running":
        s.preemptions += 1
        if s.phase == DECODE:
            s.phase = PREFILL
    w.policy.on_evicted(sid)
    return n
