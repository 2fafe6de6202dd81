"""The B200 drop-in (GpuMarsPolicy + balance_and_admit) produces the
reference's event log byte for byte.

Every frozen reference run (tests/golden/sim_logs.json: 12/64/80/200-session
workloads, the starvation run, the OpenHands-style heavy preset, and the
coordinator / co-scheduler / control-plane ablations) is replayed through the
reference tick order with the GPU policy and the GPU admission controller;
the SHA-256 of the JSONL log must equal the reference's.
"""

import hashlib

import pytest

from paper_2604_26963_b200.admission import balance_and_admit
from paper_2604_26963_b200.policy import GpuMarsPolicy, make_gpu_policy
from tests._sim import SIM, SIM_BASE, VARIANT_KW, run_sim

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("key", sorted(SIM))
def test_dropin_event_log_is_byte_identical(key):
    variant = key.split("/")[1]
    pol = GpuMarsPolicy(**VARIANT_KW[variant])
    out = run_sim(key, policy=pol, balance_and_admit=balance_and_admit)
    pol.close()
    data = out.log.jsonl_bytes()
    got = hashlib.sha256(data).hexdigest()
    if got != SIM[key]["sha256"]:
        import os

        os.makedirs("gpurun_out", exist_ok=True)
        with open(f"gpurun_out/dropin_{key.replace('/', '_')}.jsonl", "wb") as fh:
            fh.write(data)
    assert len(out.events) == SIM[key]["records"]
    assert got == SIM[key]["sha256"]
    assert out.counters == SIM[key]["counters"]


# every frozen comparison-policy run, demo64/program_priority's 173K-record
# log included
BASE_KEYS = sorted(SIM_BASE)


@pytest.mark.parametrize("key", BASE_KEYS)
def test_comparison_policy_event_log_is_byte_identical(key):
    """fcfs / program_priority / static_ttl / dynamic_ttl through the B200
    drop-ins reproduce the reference's own event logs byte for byte."""
    pol = make_gpu_policy(key.split("/")[1])
    out = run_sim(key, policy=pol)
    pol.close()
    assert len(out.events) == SIM_BASE[key]["records"]
    assert hashlib.sha256(out.log.jsonl_bytes()).hexdigest() == SIM_BASE[key]["sha256"]
    assert out.counters == SIM_BASE[key]["counters"]
