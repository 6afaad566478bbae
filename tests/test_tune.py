"""Autotuner host logic (paper_2406_06858_b200/tune.py) against the reference
tuner's own test cases (tests/test_tune.cpp): comm-tile halving, the knob
cross product, tie-break on the encoding, the cache file, the CSV report and
the abort-on-wrong-config rule. The device objective is replaced by a fake
here; tests/test_gpu_parity.py::test_tuner_on_device runs the real one."""
import json

import pytest

import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import tune as T

K_AG = fx.ProblemSpec(32, 8, 16, 4, fx.ALLGATHER_GEMM)  # rpr = 8 with 2x2 tiles: 3 comm sizes


def small_ag_space():
    return T.KnobSpace(gemm_tile_shapes=[fx.TileShape(2, 2)], transfer_modes=[fx.PULL, fx.PUSH],
                       swizzle_policies=[fx.SWIZZLE_NAIVE, fx.SWIZZLE_ARRIVAL_ALIGNED])


def test_comm_tile_sizes_halve_to_the_tile():  # test_tune.cpp:26-33
    assert T.comm_tile_sizes(8, 2) == [8, 4, 2]
    assert T.comm_tile_sizes(4, 4) == [4]
    assert T.comm_tile_sizes(12, 3) == [12, 6, 3]
    assert T.comm_tile_sizes(12, 4) == [12, 4]
    with pytest.raises(fx.ConfigError):
        T.comm_tile_sizes(8, 3)


def test_enumeration_cross_product():  # test_tune.cpp:35-73
    grid = T.enumerate_knobs(K_AG, small_ag_space())
    assert len(grid) == 12  # 1 tile x 2 transfers x 3 comm sizes x 2 swizzles
    assert len({c.encode() for c in grid}) == 12
    assert all(c.write == fx.FUSED_REDUCE for c in grid)
    rs = fx.ProblemSpec(32, 8, 16, 4, fx.GEMM_REDUCESCATTER)
    ks = small_ag_space()
    ks.write_modes = [fx.WRITE_ALLTOALL, fx.FUSED_REDUCE]
    ks.swizzle_policies = [fx.SWIZZLE_NAIVE, fx.SWIZZLE_RANK_SHIFTED, fx.SWIZZLE_ARRIVAL_ALIGNED]
    grid = T.enumerate_knobs(rs, ks)
    assert len(grid) == 4
    assert all(c.swizzle != fx.SWIZZLE_ARRIVAL_ALIGNED and c.rows_per_comm_tile == rs.rows_per_rank() for c in grid)
    ks = small_ag_space()
    ks.gemm_tile_shapes = [fx.TileShape(64, 64)]
    with pytest.raises(fx.ConfigError):
        T.enumerate_knobs(K_AG, ks)
    ks = small_ag_space()
    ks.comm_tile_override = [8, 5, 2]
    grid = T.enumerate_knobs(K_AG, ks)
    assert len(grid) == 8 and all(c.rows_per_comm_tile in (8, 2) for c in grid)


def test_b200_knobs_extend_the_grid():
    ks = T.default_knob_space(fx.ProblemSpec(4096, 28672, 8192, 8, fx.ALLGATHER_GEMM))
    assert ks.cta_groups == [1, 2] and ks.ag_engines == [1, 2]
    grid = T.enumerate_knobs(fx.ProblemSpec(4096, 28672, 8192, 8, fx.ALLGATHER_GEMM), ks)
    assert any(c.ag_engine == 2 and c.transfer == fx.PUSH for c in grid)  # the SM engine pulls and pushes
    assert len({c.encode() for c in grid}) == len(grid)
    assert "cta=2" in grid[-1].encode() or "cta=1" in grid[-1].encode()


def _fake(times):
    return lambda cfg: [times(cfg)] * 3


def test_tuning_picks_the_optimum_and_breaks_ties_on_encoding(tmp_path):  # test_tune.cpp:75-117
    grid = T.enumerate_knobs(K_AG, small_ag_space())
    cost = {c.encode(): 10.0 + i % 5 for i, c in enumerate(grid)}
    res = T.tune(K_AG, small_ag_space(), _fake(lambda c: cost[c.encode()]), lambda c: None, repetitions=3)
    assert res.objective_us == min(cost.values())
    tied = sorted(e for e, v in cost.items() if v == res.objective_us)
    assert res.best_config.encode() == tied[0]
    assert not res.from_cache


def test_cache_round_trip_and_invalidation(tmp_path):  # test_tune.cpp:119-137
    path = str(tmp_path / "tune_cache.json")
    f = _fake(lambda c: 5.0 + c.rows_per_comm_tile)
    first = T.tune(K_AG, small_ag_space(), f, lambda c: None, repetitions=3, cache_path=path, machine="B200,148")
    second = T.tune(K_AG, small_ag_space(), f, lambda c: None, repetitions=3, cache_path=path, machine="B200,148")
    assert second.from_cache and second.best_config == first.best_config
    assert second.objective_us == first.objective_us
    assert set(json.load(open(path))) == {"cache_key", "best_config", "objective_us"}  # reference cache format
    third = T.tune(K_AG, small_ag_space(), f, lambda c: None, repetitions=3, cache_path=path, machine="other")
    assert not third.from_cache


def test_repetitions_and_objective_are_validated():  # test_tune.cpp:139-145
    with pytest.raises(fx.ConfigError):
        T.tune(K_AG, small_ag_space(), _fake(lambda c: 1.0), lambda c: None, repetitions=2)
    with pytest.raises(fx.ConfigError):
        T.tune(K_AG, small_ag_space(), _fake(lambda c: 1.0), lambda c: None, objective="SimulatedTime")


def test_median_and_dispersion():  # test_tune.cpp:147-162
    res = T.tune(K_AG, small_ag_space(), lambda c: [3.0, 1.0, 2.0, 9.0, 2.5], lambda c: None, repetitions=5)
    e = res.table[0]
    assert e.objective_us == 2.5 and e.repetitions == 5
    assert e.dispersion == pytest.approx((9.0 - 1.0) / 2.5) and e.noisy


def test_a_wrong_config_aborts_the_pass():  # test_tune.cpp:164-171
    def verify(cfg):
        if cfg.transfer == fx.PUSH:
            raise AssertionError("mismatch")

    with pytest.raises(RuntimeError, match="tuning aborted: config"):
        T.tune(K_AG, small_ag_space(), _fake(lambda c: 1.0), verify, repetitions=3)


def test_csv_marks_exactly_one_best(tmp_path):  # test_tune.cpp:173-193
    res = T.tune(K_AG, small_ag_space(), _fake(lambda c: 1.0 + c.swizzle), lambda c: None, repetitions=3)
    path = tmp_path / "tune.csv"
    T.write_tune_csv(str(path), res)
    lines = path.read_text().splitlines()
    assert lines[0] == "config,objective_us,repetitions,dispersion,noisy,best"
    assert len(lines) == 13 and sum(l.endswith(",1") for l in lines[1:]) == 1
    T.write_tune_json(str(tmp_path / "tune.json"), res)
    assert json.load(open(tmp_path / "tune.json"))["best_config"] == res.best_config.encode()
