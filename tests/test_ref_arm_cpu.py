"""The bench's reference arm (oracle/ref_step.py) and the row sharding of a
snapshot, on CPU."""

import numpy as np
import pytest

from oracle.ref_step import RefStep, agentsched
from oracle.snapshot_step import run_step
from paper_2604_26963_b200.snapshot import F_QUEUED, snapshot_shard, snapshot_v1


@pytest.mark.parametrize("G", [1, 2, 5])
def test_snapshot_shard_partitions_rows(G):
    snap = snapshot_v1(20_000, seed=3)
    shards = [snapshot_shard(snap, G, g) for g in range(G)]
    assert sum(s.n for s in shards) == snap.n
    ranks = np.sort(np.concatenate([s.cols["rank"] for s in shards]))
    assert np.array_equal(ranks, snap.cols["rank"])
    for g, s in enumerate(shards):
        q = s.queue
        assert np.all((s.cols["flags"][q] & F_QUEUED) != 0)
        # the shard's list keeps the global list order
        glob = snap.queue[snap.queue % G == g]
        assert np.array_equal(s.cols["rank"][q], snap.cols["rank"][glob])
        held = -(-s.cols["kv"].astype(np.int64) // 16)
        assert s.total_blocks - s.free_blocks == held.sum()
        run_step(s.copy())  # a consistent table the oracle accepts


@pytest.mark.parametrize("pool", ["headroom", "pressure"])
def test_reference_arm_step_matches_oracle(pool):
    """The timed reference step makes the oracle's decisions."""
    if agentsched() is None:
        pytest.skip("baseline/_ref not installed")
    snap = snapshot_v1(8_000, seed=17, pool=pool)
    got = RefStep(snap.copy()).run()
    want = run_step(snap.copy())
    assert got["evictions"] == len(want["evictions"])
    assert got["tokens"] == want["total_tokens"]
    assert got["admitted"] == len(want["control"]["admitted"])
