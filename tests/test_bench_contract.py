"""bench.py's host-side contract pieces (CPU): the stratified step sample, the
identical `config` object of both arms, the round-robin C3 sharding and the
max/sum reduction over ranks."""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def test_sampled_steps_cover_the_trajectory_at_a_fixed_stride():
    steps = bench.sampled_steps(4381, 200, 5)
    assert len(steps) == 200 and steps == sorted(set(steps))
    assert steps[0] >= 5 and steps[-1] < 4381
    gaps = {b - a for a, b in zip(steps, steps[1:])}
    assert max(gaps) - min(gaps) <= 1                    # fixed stride
    assert steps[-1] > 4381 * 0.95 and steps[0] < 4381 * 0.05   # whole trajectory, not a window
    assert bench.sampled_steps(50, 200, 5) == list(range(5, 50))


def test_both_arms_report_the_same_config():
    args = argparse.Namespace(batch=64, threshold=2, steps=20, warmup=3)
    a = bench.workload_config(1, args)
    b = bench.workload_config(1, args)
    assert a == b and a["global_batch"] == 64 and "C2" in a["workload"]
    assert bench.workload_config(8, args)["global_batch"] == 512


def test_c3_round_robin_sharding_partitions_the_documents():
    for world in (1, 2, 4, 8):
        shards = [bench.shard_docs(r, world) for r in range(world)]
        flat = sorted(i for s in shards for i in s)
        assert flat == list(range(64 * world))
        assert all(len(s) == 64 for s in shards)
        assert all(i % world == r for r, s in enumerate(shards) for i in s)


def test_reduce_over_ranks_without_dist_is_identity():
    assert bench.reduce_over_ranks(None, [1.5, 2.5], [10, 20]) == (1.5, 2.5, 10, 20)
