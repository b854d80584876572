"""bench.py's host logic without a GPU: the workload / sharding definitions both arms share,
and the reference arm's sweep extrapolation."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1602_00412_b200 import synthetic as S  # noqa: E402


def test_default_workload_is_the_largest_single_gpu_config():
    stream, scaling, cfg = bench.workload(bench.DEFAULT_CONFIG, 1, 0)
    assert bench.DEFAULT_CONFIG == "c4" and cfg["config_index"] == 3
    assert (stream.n, stream.d, stream.ell, stream.seed) == (5_000_000, 50_000, 128, 3) and scaling == "weak"


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shards_tile_one_stream(world):
    stream, scaling, cfg = bench.workload("c4", world, 0)
    assert stream.n == world * 5_000_000 and cfg["shards"] == world
    spans = [S.shard_rows(stream.n, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == stream.n
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert all(r1 - r0 == 5_000_000 for r0, r1 in spans)  # weak scaling: a c4-sized shard per rank


def test_c5_is_configs4_split_over_the_ranks():
    stream, scaling, cfg = bench.workload("c5", 8, 0)
    assert scaling == "strong" and stream.n == 50_000_000 and cfg["config_index"] == 4
    assert S.shard_rows(stream.n, 8, 7) == (43_750_000, 50_000_000)


def test_both_arms_share_the_config_dict():
    assert bench.workload("c4", 2, 0)[2] == bench.workload("c4", 2, 0)[2]


def test_power_q_matches_the_reference_formula(oracle):
    for m in (1000, 10_000, 50_000, 100_000, 1_000_000, 250_000):
        assert bench.power_q(m) == oracle.power_iteration_count(m)


def test_sweep_extrapolation():
    # two processes, each: 1000 nnz in 2 s per sweep; c4 (q = 49): rate = nnz / ((q + 1) t)
    nnz_s, rows_s = bench.sweep_rate("c4", [(2.0, 1000, 100), (2.0, 1000, 100)])
    assert nnz_s == pytest.approx(2 * 1000 / (50 * 2.0)) and rows_s == pytest.approx(2 * 100 / (50 * 2.0))
