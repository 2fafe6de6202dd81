"""Runs a frozen reference trace through the oracle tick loop with any policy."""

import json
import os

from oracle import admission as oa
from oracle import loop, tracefile
from oracle import policy as op
from tests.conftest import GOLDEN

SIM = json.load(open(os.path.join(GOLDEN, "sim_logs.json")))
# the reference's comparison policies (fcfs, program_priority, static/dynamic ttl)
SIM_BASE = json.load(open(os.path.join(GOLDEN, "sim_logs_baselines.json")))
VARIANT_KW = {"mars": {}, "mars-no-coordinator": {"enable_coordinator": False},
              "mars-no-coscheduler": {"enable_coscheduler": False}, "mars-no-control": {}}


def run_sim(key, policy=None, balance_and_admit=None):
    spec = SIM[key] if key in SIM else SIM_BASE[key]
    traces = tracefile.load(os.path.join(GOLDEN, spec["trace"]))
    eng = loop.Engine(**spec["engine"])
    variant = key.split("/")[1]
    if policy is not None:
        pol = policy
    elif variant in VARIANT_KW:
        pol = op.MarsOracle(**VARIANT_KW[variant])
    else:
        pol = op.make_oracle_policy(variant)
    run = dict(spec["run"])
    if "controller" in run:
        run["controller"] = oa.Controller(**run["controller"])
    return loop.run(traces, eng, pol, balance_and_admit=balance_and_admit, **run)
