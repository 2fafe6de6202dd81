"""Block-ID restatement of the reference pool.

The reference ``KvPool`` (agentsched/engine.py:116-221) counts blocks only.
The B200 KV manager hands out concrete block IDs; this is the written-down
policy it follows, as a deliberately literal CPU oracle that replays the
reference's own pool op stream (the ``KvPool.observer`` callbacks,
engine.py:129-143, in ``seq`` order):

* a LIFO free stack whose pops initially yield 0, 1, 2, ...;
* ``alloc(sid, n)``: pop ``n`` IDs, append them to ``sid``'s table in pop order;
* ``free(sid, n)`` (also ``free`` with ``from_pinned``, i.e. release_pinned):
  remove the LAST ``n`` IDs of the table and push them in reverse table order
  (last ID first), so the first removed ID ends on top and an immediate
  re-allocation returns the same IDs in the same order;
* ``pin`` / ``unpin``: ownership moves, the table is untouched.

TEST INFRASTRUCTURE ONLY.
"""

from __future__ import annotations

from typing import Dict, List


class BlockIdPool:
    def __init__(self, total: int) -> None:
        self.total = total
        self.stack: List[int] = list(range(total - 1, -1, -1))  # top = last element
        self.tables: Dict[str, List[int]] = {}
        self.pinned: Dict[str, bool] = {}

    def alloc(self, sid: str, n: int) -> None:
        if n > len(self.stack):
            raise RuntimeError("block pool exhausted")
        t = self.tables.setdefault(sid, [])
        for _ in range(n):
            t.append(self.stack.pop())

    def free(self, sid: str, n: int) -> None:
        t = self.tables[sid]
        if n > len(t):
            raise RuntimeError(f"{sid} holds {len(t)} blocks, not {n}")
        for _ in range(n):
            self.stack.append(t.pop())
        if not t:
            del self.tables[sid]
            self.pinned.pop(sid, None)

    def apply(self, op: str, sid: str, n: int, from_pinned: bool = False) -> None:
        if op == "alloc":
            self.alloc(sid, n)
        elif op == "free":
            self.free(sid, n)
        elif op == "pin":
            self.pinned[sid] = True
        elif op == "unpin":
            self.pinned.pop(sid, None)
        else:
            raise ValueError(op)

    def table(self, sid: str) -> List[int]:
        return list(self.tables.get(sid, []))

    def top(self, k: int) -> List[int]:
        """The next k IDs pops would return."""
        return self.stack[::-1][:k]
