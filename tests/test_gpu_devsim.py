"""A whole frozen reference trace with the tick on the device
(paper_2604_26963_b200.devsim): the scheduling
half, the tick's tail and resume_from_tool all run as device kernels, the
host keeps arrivals, the tool plane and the idle-tick jump.  The run
counters (admissions, completions, evictions, preemptions, warm / cold
resumes, pins, GPU tokens) and the final clock must equal the reference's
own run of the same trace (tests/golden/sim_logs.json)."""

import os

import pytest

from oracle import tracefile
from paper_2604_26963_b200.devsim import run_device_simulation
from tests._sim import SIM, VARIANT_KW
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

# the device loop runs MARS with its control plane (mars-no-control admits at
# arrival, outside the device control plane; starvation runs without it)
KEYS = sorted(k for k in SIM if not k.endswith("no-control") and not k.startswith("starvation"))


@pytest.mark.parametrize("key", KEYS)
def test_device_simulation_reproduces_reference_counters(key):
    spec = SIM[key]
    traces = tracefile.load(os.path.join(GOLDEN, spec["trace"]))
    kw = dict(VARIANT_KW[key.split("/")[1]])
    ctl = spec["run"].get("controller") or {}
    cnt, horizon = run_device_simulation(traces, spec["engine"]["total_blocks"],
                                         spec["engine"]["tool_worker_slots"],
                                         initial_window=ctl.get("initial_window"), **kw)
    assert cnt == spec["counters"]
    assert horizon == spec["horizon_s"]
