"""The block-ID restatement itself (CPU): LIFO policy and conservation."""

import random

from oracle.block_ids import BlockIdPool


def test_pops_start_at_zero_and_free_returns_the_same_ids():
    p = BlockIdPool(10)
    p.alloc("a", 3)
    p.alloc("b", 2)
    assert p.table("a") == [0, 1, 2] and p.table("b") == [3, 4]
    p.free("a", 3)
    assert p.top(4) == [0, 1, 2, 5]
    p.alloc("c", 2)
    assert p.table("c") == [0, 1]


def test_partial_free_releases_the_tail():
    p = BlockIdPool(8)
    p.alloc("a", 5)
    p.free("a", 2)
    assert p.table("a") == [0, 1, 2] and p.top(3) == [3, 4, 5]


def test_conservation_under_a_random_op_stream():
    rng = random.Random(5)
    p = BlockIdPool(300)
    live = {}
    for i in range(5000):
        if live and rng.random() < 0.45:
            sid = rng.choice(sorted(live))
            n = rng.randrange(1, live[sid] + 1)
            p.free(sid, n)
            live[sid] -= n
            if not live[sid]:
                del live[sid]
        else:
            n = rng.randrange(1, 20)
            if n <= len(p.stack):
                sid = f"s{rng.randrange(40)}"
                p.alloc(sid, n)
                live[sid] = live.get(sid, 0) + n
        ids = [b for t in p.tables.values() for b in t] + p.stack
        assert sorted(ids) == list(range(300))
