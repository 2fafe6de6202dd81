"""A whole frozen reference trace with the tick on the device
(paper_2604_26963_b200.devsim): the scheduling
half, the tick's tail and resume_from_tool all run as device kernels, the
host keeps arrivals, the tool plane and the idle-tick jump.  The run
counters (admissions, completions, evictions, preemptions, warm / cold
resumes, pins, GPU tokens), the final clock and the event log's bytes
(SHA-256 over the JSONL) must equal the reference's own
run of the same trace (tests/golden/sim_logs.json)."""

import hashlib
import json
import os

import pytest

from oracle import tracefile
from paper_2604_26963_b200.devsim import EventLog, run_device_simulation
from tests._sim import SIM, SIM_BASE, VARIANT_KW, run_sim
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _check_log(key, spec, log):
    data = log.jsonl_bytes()
    if len(log.records) == spec["records"] and \
            hashlib.sha256(data).hexdigest() == spec["sha256"]:
        return
    # locate the first record that differs from the oracle's run (itself
    # pinned to the same digests by tests/test_oracle_golden.py)
    ref = run_sim(key).events
    for i, (a, b) in enumerate(zip(log.records, ref)):
        if json.dumps(a, separators=(",", ":")) != json.dumps(b, separators=(",", ":")):
            ctx = "\n".join(json.dumps(r) for r in ref[max(0, i - 3):i])
            pytest.fail(f"record {i + 1} differs\n  device: {json.dumps(a)}\n"
                        f"  reference: {json.dumps(b)}\n  after:\n{ctx}")
    pytest.fail(f"{len(log.records)} records, the reference has {len(ref)}")


@pytest.mark.parametrize("key", sorted(SIM))
def test_device_simulation_reproduces_reference_counters(key):
    """MARS, its ablations and the control-plane-off runs (admission at arrival)."""
    spec = SIM[key]
    traces = tracefile.load(os.path.join(GOLDEN, spec["trace"]))
    kw = dict(VARIANT_KW[key.split("/")[1]])
    ctl = spec["run"].get("controller") or {}
    log = EventLog()
    cnt, horizon = run_device_simulation(
        traces, spec["engine"]["total_blocks"], spec["engine"]["tool_worker_slots"],
        enable_control_plane=spec["run"].get("enable_control_plane", True),
        initial_window=ctl.get("initial_window"), log=log, **kw)
    assert cnt == spec["counters"]
    assert horizon == spec["horizon_s"]
    _check_log(key, spec, log)


# every frozen comparison-policy run, demo64/program_priority's 173K-record
# log included
BASE_KEYS = sorted(SIM_BASE)


@pytest.mark.parametrize("key", BASE_KEYS)
def test_device_simulation_comparison_policies(key):
    """fcfs / program_priority / static_ttl / dynamic_ttl: admission at
    arrival, their plans, boundaries and pins all on the device."""
    spec = SIM_BASE[key]
    traces = tracefile.load(os.path.join(GOLDEN, spec["trace"]))
    log = EventLog()
    cnt, horizon = run_device_simulation(traces, spec["engine"]["total_blocks"],
                                         spec["engine"]["tool_worker_slots"],
                                         policy=spec["policy"], log=log)
    assert cnt == spec["counters"]
    assert horizon == spec["horizon_s"]
    _check_log(key, spec, log)


def test_device_simulation_without_log_matches():
    """The log is optional: the same run without it gives the same counters."""
    key = "small12/mars"
    spec = SIM[key]
    traces = tracefile.load(os.path.join(GOLDEN, spec["trace"]))
    cnt, horizon = run_device_simulation(traces, spec["engine"]["total_blocks"],
                                         spec["engine"]["tool_worker_slots"])
    assert cnt == spec["counters"] and horizon == spec["horizon_s"]


@pytest.mark.parametrize("key", ["small12/mars", "small12/mars-no-control", "demo64/mars",
                                 "small12/static_ttl", "small12/fcfs"])
def test_device_simulation_block_ids(key):
    """The device block-ID manager riding along a whole device-resident run
    (plan journal, expiries, the tail's frees, return-time releases) ends
    with the free stack the block-ID restatement (oracle/block_ids.py) builds
    from the run's event log -- itself byte-identical to the reference's."""
    from oracle.block_ids import BlockIdPool
    spec = SIM[key] if key in SIM else SIM_BASE[key]
    traces = tracefile.load(os.path.join(GOLDEN, spec["trace"]))
    variant = key.split("/")[1]
    kw = dict(VARIANT_KW.get(variant, {}))
    if key in SIM_BASE:
        kw["policy"] = spec["policy"]
    log, kv = EventLog(), {}
    total = spec["engine"]["total_blocks"]
    run_device_simulation(traces, total, spec["engine"]["tool_worker_slots"],
                          enable_control_plane=spec["run"].get("enable_control_plane", True),
                          log=log, kv_state=kv, **kw)
    _check_log(key, spec, log)
    pool = BlockIdPool(total)
    n_ops = 0
    for r in log.records:
        if r["kind"] in ("alloc", "free", "pin", "unpin"):
            pool.apply(r["kind"], r["session_id"], r["blocks"], r.get("from_pinned", False))
            n_ops += 1
    assert n_ops > 100
    assert kv["status"] == 0
    assert kv["top"].tolist() == pool.top(total)


def _synthetic(n, seed):
    """A larger seeded trace than the frozen ones: many sessions arriving
    together into a tight pool, so preemptions, reclaims, pins and their
    expiries all happen often."""
    import numpy as np
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        k = int(rng.integers(1, 5))
        rounds = []
        for j in range(k):
            tool = None if j == k - 1 else float(np.round(rng.uniform(0.05, 6.0), 3))
            rounds.append(tracefile.RoundRec(int(rng.integers(100, 5000)),
                                             int(rng.integers(1, 160)), tool))
        out.append(tracefile.Trace(f"syn{i:04d}", float(np.round(rng.uniform(0, 15.0), 3)),
                                   rounds))
    return out


SYN = {  # label: (policy, MARS switches, control plane, sessions, pool blocks, tool slots)
    "mars": ("mars", {}, True, 160, 2500, 6),
    "mars-600": ("mars", {}, True, 600, 6000, 16),
    "mars-no-coordinator": ("mars", {"enable_coordinator": False}, True, 150, 2400, 6),
    "mars-no-coscheduler": ("mars", {"enable_coscheduler": False}, True, 150, 2400, 6),
    "mars-no-control": ("mars", {}, False, 120, 2000, 4),
    "fcfs": ("fcfs", {}, True, 100, 2200, 4),
    "program_priority": ("program_priority", {}, True, 100, 2200, 4),
    "static_ttl": ("static_ttl", {}, True, 120, 2000, 4),
    "dynamic_ttl": ("dynamic_ttl", {}, True, 120, 2000, 4),
}


@pytest.mark.parametrize("label", sorted(SYN))
def test_device_simulation_synthetic_matches_oracle(label):
    """Whole device-resident run of a synthetic trace against the oracle's
    tick loop (oracle/loop.py, itself pinned to the reference's logs):
    counters, final clock, the event log byte for byte and the block IDs."""
    from oracle import loop
    from oracle import policy as op
    from oracle.block_ids import BlockIdPool
    kind, sw, ctl_on, n, blocks, slots = SYN[label]
    traces = _synthetic(n, seed=n + blocks)
    pol = op.MarsOracle(**sw) if kind == "mars" else op.make_oracle_policy(kind)
    ref = loop.run(traces, loop.Engine(blocks, tool_worker_slots=slots), pol,
                   enable_control_plane=ctl_on)
    assert ref.counters["preemptions"] > 0 and ref.counters["completed"] == n
    log, kv = EventLog(), {}
    cnt, horizon = run_device_simulation(traces, blocks, slots, policy=kind,
                                         enable_control_plane=ctl_on, log=log, kv_state=kv,
                                         **sw)
    assert cnt == ref.counters
    assert horizon == ref.horizon_s
    got, want = log.jsonl_bytes(), ref.log.jsonl_bytes()
    if got != want:
        for i, (a, b) in enumerate(zip(log.records, ref.events)):
            if json.dumps(a) != json.dumps(b):
                pytest.fail(f"record {i + 1} differs\n  device: {json.dumps(a)}\n"
                            f"  oracle: {json.dumps(b)}")
        pytest.fail(f"{len(log.records)} records, the oracle has {len(ref.events)}")
    pool = BlockIdPool(blocks)
    for r in log.records:
        if r["kind"] in ("alloc", "free", "pin", "unpin"):
            pool.apply(r["kind"], r["session_id"], r["blocks"], r.get("from_pinned", False))
    assert kv["status"] == 0 and kv["top"].tolist() == pool.top(blocks)
