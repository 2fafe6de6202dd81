"""Frozen session traces: JSONL records in the reference's wire format
(``agentsched/workload.py:276-330``).  TEST INFRASTRUCTURE ONLY.

Parity traces are generated once by the reference (``oracle/make_golden.py``)
and committed, so they do not depend on numpy/scipy versions on the box.
"""

from __future__ import annotations

import json
from typing import List, Optional, Sequence


class RoundRec:
    __slots__ = ("new_prefill_tokens", "decode_tokens", "tool_duration_s")

    def __init__(self, new_prefill_tokens: int, decode_tokens: int,
                 tool_duration_s: Optional[float]) -> None:
        self.new_prefill_tokens = new_prefill_tokens
        self.decode_tokens = decode_tokens
        self.tool_duration_s = tool_duration_s


class Trace:
    __slots__ = ("session_id", "arrival_time_s", "rounds")

    def __init__(self, session_id: str, arrival_time_s: float, rounds: Sequence[RoundRec]) -> None:
        self.session_id = session_id
        self.arrival_time_s = arrival_time_s
        self.rounds = tuple(rounds)

    @property
    def total_context_tokens(self) -> int:
        return sum(r.new_prefill_tokens + r.decode_tokens for r in self.rounds)


def loads(text: str) -> List[Trace]:
    out = []
    for line in text.splitlines():
        line = line.strip()
        if not line:
            continue
        rec = json.loads(line)
        out.append(Trace(str(rec["session_id"]), float(rec["arrival_time_s"]),
                         [RoundRec(int(r["new_prefill_tokens"]), int(r["decode_tokens"]),
                                   None if r["tool_duration_s"] is None else float(r["tool_duration_s"]))
                          for r in rec["rounds"]]))
    return out


def load(path: str) -> List[Trace]:
    with open(path, "r", encoding="utf-8") as fh:
        return loads(fh.read())


def dumps(traces) -> str:
    lines = []
    for t in traces:
        lines.append(json.dumps({
            "session_id": t.session_id,
            "arrival_time_s": t.arrival_time_s,
            "rounds": [{"new_prefill_tokens": r.new_prefill_tokens,
                        "decode_tokens": r.decode_tokens,
                        "tool_duration_s": r.tool_duration_s} for r in t.rounds],
        }, separators=(",", ":")))
    return "\n".join(lines) + "\n"
