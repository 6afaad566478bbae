"""Host logic of the product, through the C ABI, without a GPU.

Mirrors the reference's test_swizzle.cpp / test_core.cpp / test_engine.cpp
host-side cases: validation rules and messages (problem.cpp:15-38), grid_for,
tile_order for every swizzle kind against the reference's own output
(swizzle.cpp:23-80), comm order (topology.cpp:102-178) and make_comm_specs
with CommTileSpec::validate (engine.cpp:40-99).
"""
import json
import os

import pytest

import paper_2406_06858_b200 as fx

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_ref.json")


def _doc():
    with open(GOLDEN) as f:
        return json.load(f)


AG, RS = fx.ALLGATHER_GEMM, fx.GEMM_REDUCESCATTER


def test_problem_validation_rules_and_messages():
    fx.ProblemSpec(16, 16, 16, 4, AG).validate()
    with pytest.raises(fx.ConfigError, match="positive"):
        fx.ProblemSpec(0, 16, 16, 4, AG).validate()
    with pytest.raises(fx.ConfigError, match="tp must be positive"):
        fx.ProblemSpec(16, 16, 16, 0, AG).validate()
    with pytest.raises(fx.ConfigError, match="m=10 not divisible by tp=4"):
        fx.ProblemSpec(10, 16, 16, 4, AG).validate()
    with pytest.raises(fx.ConfigError, match="AllGatherGemm requires n divisible by tp"):
        fx.ProblemSpec(16, 10, 16, 4, AG).validate()
    with pytest.raises(fx.ConfigError, match="GemmReduceScatter requires k divisible by tp"):
        fx.ProblemSpec(16, 16, 10, 4, RS).validate()


def test_tiling_rules():
    p = fx.ProblemSpec(16, 16, 16, 4, AG)
    fx.validate_tiling(p, fx.TileShape(2, 2))
    with pytest.raises(fx.ConfigError, match="tm=3 must divide m/tp=4"):
        fx.validate_tiling(p, fx.TileShape(3, 2))
    with pytest.raises(fx.ConfigError, match="tm=8 must divide m/tp=4"):
        fx.validate_tiling(p, fx.TileShape(8, 2))
    with pytest.raises(fx.ConfigError, match="tn=3 must divide the local output cols=4"):
        fx.validate_tiling(p, fx.TileShape(2, 3))
    with pytest.raises(fx.ConfigError, match="positive"):
        fx.validate_tiling(p, fx.TileShape(0, 2))
    assert fx.grid_for(p, fx.TileShape(2, 2)) == (8, 2, 4)
    assert fx.grid_for(fx.ProblemSpec(16, 16, 16, 4, RS), fx.TileShape(2, 4)) == (8, 4, 4)


def test_tile_order_matches_reference_for_every_kind():
    cases = _doc()["tile_orders"]
    assert len(cases) > 50
    for c in cases:
        p = fx.ProblemSpec(c["m"], c["n"], c["k"], c["tp"], c["pattern"])
        got = fx.tile_order(p, fx.TileShape(c["tm"], c["tn"]), c["kind"], c["rank"], c["shift"])
        assert got == [tuple(x) for x in c["order"]], c


def test_rank_shifted_and_arrival_aligned_block_orders():
    """test_swizzle.cpp:44-56."""
    p = fx.ProblemSpec(4, 4, 4, 4, RS)  # one tile row per block, one column
    blocks = [r for r, _ in fx.tile_order(p, fx.TileShape(1, 4), fx.SWIZZLE_RANK_SHIFTED, 1)]
    assert blocks == [2, 3, 0, 1]
    p = fx.ProblemSpec(8, 8, 8, 8, AG)
    blocks = [r for r, _ in fx.tile_order(p, fx.TileShape(1, 1), fx.SWIZZLE_ARRIVAL_ALIGNED, 5)]
    assert blocks == [5, 6, 7, 0, 1, 2, 3, 4]
    naive = fx.tile_order(fx.ProblemSpec(4, 8, 4, 2, AG), fx.TileShape(2, 2), fx.SWIZZLE_NAIVE, 0)
    assert naive == [(0, 0), (0, 1), (1, 0), (1, 1)]


@pytest.mark.parametrize("kind", [fx.SWIZZLE_NAIVE, fx.SWIZZLE_RANK_SHIFTED, fx.SWIZZLE_ARRIVAL_ALIGNED])
def test_tile_order_is_a_bijection(kind):
    """test_swizzle.cpp:65-93 (every kind is a bijection on the grid)."""
    for tp in (1, 2, 4, 8):
        for rpb in (1, 2, 3):
            for cols in (1, 3, 8):
                m, tm = tp * rpb * 2, 2
                p = fx.ProblemSpec(m, cols * tp, 4, tp, AG)
                for rank in range(tp):
                    order = fx.tile_order(p, fx.TileShape(tm, 1), kind, rank)
                    assert sorted(order) == [(r, c) for r in range(m // tm) for c in range(cols)]


def test_rank_shifted_is_contention_free():
    """test_swizzle.cpp:95-108: at every step the ranks target distinct blocks."""
    tp = 8
    p = fx.ProblemSpec(8 * tp, 8, 8 * tp, tp, RS)
    orders = [fx.tile_order(p, fx.TileShape(8, 8), fx.SWIZZLE_RANK_SHIFTED, r) for r in range(tp)]
    for step in range(tp):
        assert len({orders[r][step][0] // 1 for r in range(tp)}) == tp


def test_ring_comm_order():
    """test_swizzle.cpp:110-115: rank 5 of 8 pulls 6, 7, 0, ..., 4."""
    order = fx.comm_order(5, 8, 4, 4)
    assert [p for p, _, _ in order] == [6, 7, 0, 1, 2, 3, 4]
    assert [b for _, b, _ in order] == [24, 28, 0, 4, 8, 12, 16]
    halved = fx.comm_order(1, 2, 8, 2)
    assert halved == [(0, 0, 2), (0, 2, 2), (0, 4, 2), (0, 6, 2)]
    with pytest.raises(fx.ConfigError):
        fx.comm_order(0, 2, 8, 3)


def test_make_comm_spec_matches_reference():
    for c in _doc()["comm_specs"]:
        p = fx.ProblemSpec(c["m"], c["n"], c["k"], c["tp"], c["pattern"])
        got = fx.make_comm_spec(p, c["rank"], c["rpct"], c["transfer"])
        assert got == [tuple(x) for x in c["order"]], c


def test_make_comm_spec_rejects_bad_comm_tiles():
    p = fx.ProblemSpec(16, 16, 16, 4, AG)
    with pytest.raises(fx.ConfigError, match="rows_per_comm_tile=3 must divide"):
        fx.make_comm_spec(p, 0, 3, fx.PULL)
    with pytest.raises(fx.ConfigError):
        fx.make_comm_spec(p, 4, 2, fx.PULL)


def test_push_spec_carries_local_tiles_to_every_peer():
    p = fx.ProblemSpec(32, 16, 16, 4, AG)
    spec = fx.make_comm_spec(p, 2, 4, fx.PUSH)
    assert len(spec) == 3 * 2
    assert {peer for peer, _, _ in spec} == {3, 0, 1}
    assert all(16 <= b < 24 for _, b, _ in spec)
