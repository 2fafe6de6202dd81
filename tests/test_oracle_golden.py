"""Pins the CPU oracle against fixtures frozen from the reference itself.

Everything here runs on CPU.  The fixtures were produced by
``oracle/make_golden.py`` from ``/root/reference`` (the reference package is
not needed to run these tests).
"""

import hashlib
import json
import os

import pytest

from oracle import admission as oa
from oracle import core as oc
from oracle import loop, tracefile
from oracle import policy as op
from oracle.snapshot_step import run_step
from paper_2604_26963_b200.snapshot import snapshot_v1
from tests._canon import canon

from tests.conftest import GOLDEN


def _load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


SIM = _load("sim_logs.json")
SNAP = _load("snapshot_steps.json")
KAT = _load("kat.json")

from tests._sim import SIM_BASE
from tests._sim import run_sim as run_oracle_sim


@pytest.mark.parametrize("key", sorted(SIM))
def test_oracle_sim_log_is_byte_identical_to_reference(key):
    out = run_oracle_sim(key)
    got = hashlib.sha256(out.log.jsonl_bytes()).hexdigest()
    assert len(out.events) == SIM[key]["records"]
    assert got == SIM[key]["sha256"]
    assert out.counters == SIM[key]["counters"]


@pytest.mark.parametrize("key", sorted(SIM_BASE))
def test_oracle_baseline_policy_log_is_byte_identical_to_reference(key):
    out = run_oracle_sim(key)
    assert len(out.events) == SIM_BASE[key]["records"]
    assert hashlib.sha256(out.log.jsonl_bytes()).hexdigest() == SIM_BASE[key]["sha256"]
    assert out.counters == SIM_BASE[key]["counters"]


@pytest.mark.parametrize("i", range(len(SNAP)))
def test_oracle_snapshot_step_matches_reference(i):
    case = dict(SNAP[i]["case"])
    kw = {k: case.pop(k) for k in ("enable_coordinator", "enable_coscheduler") if k in case}
    snap = snapshot_v1(case["n"], seed=case["seed"], pool=case["pool"])
    got = canon(run_step(snap, **kw))
    want = SNAP[i]["out"]
    for k in want:
        assert got[k] == want[k], k


def test_kat_retention():
    for r in KAT["retention"]:
        s = oc.Session("x", [oc.Round(1, 1)], 0.0)
        s.context_tokens, s.kv_tokens = r["ctx"], r["kv"]
        t = oa.Counters(r["total"])
        t.kv_usage_ratio = r["usage"]
        t.ema_tool_duration = r["ema"]
        d = op.retention(s, t, oc.BlockCounter(r["total"]), oc.TickModel(), op.Retention(),
                         oa.Pressure(), r["now"])
        assert (d.pin, d.benefit_s, d.cost_s, d.retention_deadline) == (
            r["pin"], r["benefit"], r["cost"], r["deadline"])


def test_kat_try_fit():
    for r in KAT["try_fit"]:
        held = oc.ceil_div(r["kv"], 16)
        pool = oc.BlockCounter(held + r["free"] + 1)
        pool.allocate("other", 1)
        if held:
            pool.allocate("self", held)
        s = oc.Session("self", [oc.Round(1, 1)], 0.0)
        s.kv_tokens = s.context_tokens = r["kv"]
        assert op.fit_chunk(s, r["desired"], pool, 16) == r["grant"]


def test_kat_pack():
    for r in KAT["pack"]:
        t = oa.Counters(10_000)
        t.cpu_overloaded = r["cpu"]
        t.available_kv = r["avail"]
        q = [oa.Pending(oc.Session(f"q{i:03d}", [oc.Round(1, 1)], 0.0), b, lg, 0.0)
             for i, (b, lg) in enumerate(zip(r["reqs"], r["longs"]))]
        assert [int(e.call.session_id[1:]) for e in oa.pack(q, t)] == r["order"]


def test_kat_admission_replay():
    t = oa.Counters(50_000)
    c = oa.Controller()
    p = oa.Pressure()
    for s in KAT["admit_replay"]:
        t.active_tools, t.queued_tools = s["active_tools"], s["queued_tools"]
        t.kv_usage_ratio, t.available_kv, t.active_sessions = s["usage"], s["avail"], s["active"]
        t.ema_blocks_per_session = s["ema_blocks"]
        oa.refresh_pressure(t, p, 8)
        assert (t.cpu_overloaded, t.kv_overloaded) == (s["cpu"], s["kvo"])
        q = [oa.Pending(oc.Session(f"q{k:03d}", [oc.Round(1, 1)], 0.0), b, False, 0.0)
             for k, b in enumerate(s["reqs"])]
        got = oa.admit_step(q, c, t, 8, p, s["now"])
        assert c.w_adm == s["w"]
        assert [int(e.call.session_id[1:]) for e in got] == s["admitted"]
        assert t.blocks_seed == s["seed"]


def test_kat_reclaim():
    for r in KAT["reclaim"]:
        pool = oc.BlockCounter(100_000)
        pool.allocate("fill", 100_000 - r["free"])
        pins = {sid: op.Pin(sid, b, 0.0, 0.0, dl, lv) for sid, b, dl, lv in r["pins"]}
        run, lv = [], {}
        for sid, kv, level in r["running"]:
            s = oc.Session(sid, [oc.Round(1, 1)], 0.0)
            s.kv_tokens = kv
            run.append(s)
            lv[sid] = level
        vs = op.choose_victims(r["need"], pool, pins, run, lambda s: lv[s.session_id], r["now"])
        assert [list(v.as_tuple()) for v in vs] == r["victims"]


def test_kat_levels_and_charges():
    m = op.Mlfq()
    for tokens, level in KAT["initial_level"]:
        assert op.level_for(tokens, m) == level
    for r in KAT["charge"]:
        st = op.Prio(r["start"], 0)
        for ch in r["charges"]:
            op.charge(st, ch, m)
        assert (st.level, st.served_tokens_at_level) == (r["level"], r["served"])


HEAVY = _load("heavy_steps.json")


@pytest.mark.parametrize("i", range(len(HEAVY)))
def test_oracle_heavy_step_matches_reference(i):
    """Heavy reclaim (dozens of victims, every policy) and tick-gridded ties:
    the oracle against the reference's own step (oracle/make_golden.py
    --only heavy)."""
    from oracle.make_golden import heavy_kw, heavy_snapshot

    case = HEAVY[i]["case"]
    got = canon(run_step(heavy_snapshot(case), **heavy_kw(case)))
    for k, v in HEAVY[i]["out"].items():
        assert got[k] == v, k
