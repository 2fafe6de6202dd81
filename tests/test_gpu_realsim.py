"""The drop-ins inside the reference's OWN loop: ``agentsched.sim.run_simulation``
(sim.py:90-431) from the unmodified reference package (baseline/_ref), with the
INTEGRATION.md binding applied -- the GPU policy built the way the
``mars_gpu`` branch of ``make_policy`` builds it (baselines.py:458-495) and
``sim.balance_and_admit`` swapped for the B200 one (sim.py:29).  The event
log must equal the reference's frozen log byte for byte, and -- for engine
parameters no frozen run uses (a non-default GpuModel) -- the log of the
reference's own MarsPolicy run live in the same process."""

import hashlib
import json
import os

import pytest

from tests.conftest import GOLDEN
from tests._sim import SIM, SIM_BASE, VARIANT_KW

pytestmark = pytest.mark.gpu

A = pytest.importorskip("agentsched", reason="the reference package (baseline/_ref) is not installed")
from agentsched import baselines, control, scheduler, sim, telemetry, workload  # noqa: E402

from paper_2604_26963_b200.admission import balance_and_admit as gpu_balance_and_admit  # noqa: E402
from paper_2604_26963_b200.policy import GpuMarsPolicy, make_gpu_policy  # noqa: E402


def _jsonl(events) -> bytes:
    return b"".join(json.dumps(r, separators=(",", ":")).encode() + b"\n" for r in events)


def _make(kind, gpu, variant_kw):
    """make_policy (baselines.py:458-495) with the INTEGRATION.md §1 branch."""
    mlfq, ret, pr = scheduler.MlfqConfig(), scheduler.RetentionConfig(), telemetry.PressureConfig()
    if not gpu:
        return baselines.make_policy(kind, mlfq, ret, pr, **variant_kw)
    if kind == "mars":
        return GpuMarsPolicy(mlfq, ret, pr, **variant_kw)
    return make_gpu_policy(kind, mlfq, ret, pr)


def run_real(key, gpu: bool, engine_over=None):
    spec = SIM[key] if key in SIM else SIM_BASE[key]
    traces = workload.load_trace(os.path.join(GOLDEN, spec["trace"]))
    params = sim.EngineParams(**spec["engine"], **(engine_over or {}))
    run = dict(spec["run"])
    if "controller" in run:
        run["controller"] = control.ControllerConfig(**run["controller"])
    variant = key.split("/")[1]
    kind = "mars" if variant in VARIANT_KW else variant
    pol = _make(kind, gpu, VARIANT_KW.get(variant, {}))
    if gpu:
        assert isinstance(pol, baselines.PolicyBase)
    orig = sim.balance_and_admit
    if gpu:
        sim.balance_and_admit = gpu_balance_and_admit
    try:
        res = sim.run_simulation(traces, params, pol, **run)
    finally:
        sim.balance_and_admit = orig
        if gpu:
            pol.close()
    return res


KEYS = ["small12/mars", "small12/mars-no-control", "demo64/mars", "demo64/mars-no-coordinator",
        "crit7_80/mars-no-coscheduler", "faceoff200/mars", "openhands_heavy40/mars",
        "starvation/mars"]


@pytest.mark.parametrize("key", KEYS)
def test_real_run_simulation_log_is_byte_identical(key):
    res = run_real(key, gpu=True)
    data = _jsonl(res.events)
    assert len(res.events) == SIM[key]["records"]
    assert hashlib.sha256(data).hexdigest() == SIM[key]["sha256"]
    assert res.counters == SIM[key]["counters"]


@pytest.mark.parametrize("key", ["small12/fcfs", "small12/program_priority", "small12/static_ttl",
                                 "crit7_80/dynamic_ttl", "faceoff200/fcfs"])
def test_real_run_simulation_comparison_policies(key):
    res = run_real(key, gpu=True)
    assert hashlib.sha256(_jsonl(res.events)).hexdigest() == SIM_BASE[key]["sha256"]
    assert res.counters == SIM_BASE[key]["counters"]


@pytest.mark.parametrize("key,over", [
    ("small12/mars", {"token_budget_per_tick": 256, "tick_duration_s": 0.05}),
    ("demo64/mars", {"token_budget_per_tick": 1024}),
    ("crit7_80/mars-no-coordinator", {"tick_duration_s": 0.1}),
])
def test_real_run_simulation_non_default_gpu_model(key, over):
    """A GpuModel other than the default (the engine parameters
    arrive with the first plan_tick, after registrations): the drop-in's log
    equals the reference MarsPolicy's own log for the same parameters."""
    want = run_real(key, gpu=False, engine_over=over)
    got = run_real(key, gpu=True, engine_over=over)
    assert len(got.events) == len(want.events)
    assert _jsonl(got.events) == _jsonl(want.events)
    assert got.counters == want.counters
