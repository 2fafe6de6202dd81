"""The product's trace-file reader (devsim.load_trace) reads the frozen
reference traces exactly as the oracle's reader does (CPU)."""

import os

import pytest

from oracle import tracefile
from paper_2604_26963_b200.devsim import load_trace
from tests.conftest import GOLDEN

TRACES = sorted(os.listdir(os.path.join(GOLDEN, "traces")))


@pytest.mark.parametrize("name", TRACES)
def test_load_trace_matches_the_oracle_reader(name):
    path = os.path.join(GOLDEN, "traces", name)
    got = load_trace(path)
    want = tracefile.load(path)
    assert [(t.session_id, t.arrival_time_s, [tuple(r) for r in t.rounds]) for t in got] == \
        [(t.session_id, t.arrival_time_s,
          [(r.new_prefill_tokens, r.decode_tokens, r.tool_duration_s) for r in t.rounds])
         for t in want]
