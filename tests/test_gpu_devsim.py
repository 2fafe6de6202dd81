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


# demo64/program_priority's run is ~10x longer than the others (see test_gpu_dropin)
BASE_KEYS = sorted(k for k in SIM_BASE if k != "demo64/program_priority")


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
