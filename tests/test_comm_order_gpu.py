"""The caller's comm specs (run_fused_allgather_gemm's comm_specs argument,
engine.hpp:107-111): the copy-engine transfer loop walks each rank's order
(engine.cpp:367-423) and records a TransferRecord per descriptor with device
times (CUDA events on the copy stream), copy_done <= flag_set
(test_engine.cpp:102-115); the in-kernel engine follows the arrival order the
caller's order implies. The device event trace exports to the Chrome trace
format (sim.cpp:597-610)."""
import json

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_2406_06858_b200 as fx  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import gpu_harness as H  # noqa: E402

AG = fx.ALLGATHER_GEMM


def _reversed_pull_orders(p, rpct):
    """A valid Pull spec per rank that is NOT the NVLinkRing order: peers in
    descending distance, each peer's comm tiles last-to-first."""
    rpr = p.rows_per_rank()
    orders = []
    for r in range(p.tp):
        o = []
        for d in range(p.tp - 1, 0, -1):
            q = (r + d) % p.tp
            for off in range(rpr - rpct, -1, -rpct):
                o.append((q, q * rpr + off, rpct))
        orders.append(o)
    return orders


@pytest.mark.parametrize("transfer", [fx.PULL, fx.PUSH])
def test_caller_comm_order_is_walked_and_recorded(transfer):
    p = fx.ProblemSpec(512, 512, 256, 4, AG)
    rpct = 64
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=21)
        if transfer == fx.PULL:
            orders = _reversed_pull_orders(p, rpct)
        else:  # the reference push spec with its peers reversed
            orders = [list(reversed(fx.make_comm_spec(p, r, rpct, fx.PUSH))) for r in range(p.tp)]
        assert orders[1] != fx.make_comm_spec(p, 1, rpct, transfer)
        # in-kernel engine on the same orders: correct results
        comm.ag_gemm_ordered(p, fx.TileShape(p.rows_per_rank(), p.local_cols()), orders, rpct, transfer, True,
                             fx.default_opts(out_dtype=fx.F32, ag_engine=2, wall_budget_s=5.0))
        comm.sync()
        want0 = O.dense_oracle(AG, p.m, p.n, p.k, p.tp, a, b)
        for r, g in enumerate(H.outputs(comm, p, True)):
            assert O.max_rel_error(g, want0[r]) <= H.tol(True, p.k)
        opts = fx.default_opts(out_dtype=fx.F32, ag_engine=1, trace=1, wall_budget_s=5.0)
        comm.ag_gemm_ordered(p, fx.TileShape(p.rows_per_rank(), p.local_cols()), orders, rpct, transfer, True, opts)
        comm.sync()
        want = O.dense_oracle(AG, p.m, p.n, p.k, p.tp, a, b)
        got = H.outputs(comm, p, True)
        for r in range(p.tp):
            assert O.max_rel_error(got[r], want[r]) <= H.tol(True, p.k)
        for r in range(p.tp):
            recs = comm.transfer_log(r)
            assert len(recs) == len(orders[r])
            if transfer == fx.PULL:  # issued in exactly the caller's order
                assert [(x["peer"], x["row_begin"], x["rows"]) for x in recs] == orders[r]
            else:
                assert sorted((x["peer"], x["row_begin"], x["rows"]) for x in recs) == sorted(orders[r])
            for x in recs:
                assert 0 <= x["copy_done_ns"] <= x["flag_set_ns"], x


def test_invalid_caller_orders_rejected():
    p = fx.ProblemSpec(512, 512, 256, 4, AG)
    rpct = 128
    with H.make_comm(p) as comm:
        H.upload(comm, p, seed=22)
        tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
        good = [fx.make_comm_spec(p, r, rpct, fx.PULL) for r in range(p.tp)]
        dup = [list(o) for o in good]
        dup[2][1] = dup[2][0]  # comm tile covered twice, another never
        with pytest.raises(fx.ConfigError, match="exactly once"):
            comm.ag_gemm_ordered(p, tile, dup, rpct, fx.PULL)
        wrong = [list(o) for o in good]
        q, rb, rows = wrong[0][0]
        wrong[0][0] = ((q + 1) % p.tp if (q + 1) % p.tp != 0 else 2, rb, rows)  # not the owner of those rows
        with pytest.raises(fx.BoundsError):
            comm.ag_gemm_ordered(p, tile, wrong, rpct, fx.PULL)
        comm.ag_gemm_ordered(p, tile, good, rpct, fx.PULL)  # the reference order still works
        comm.sync()


def test_chrome_trace_round_trip(tmp_path):
    p = fx.ProblemSpec(2048, 512, 512, 8, fx.GEMM_REDUCESCATTER)
    with H.make_comm(p) as comm:
        H.upload(comm, p, seed=23)
        comm.gemm_rs(p, fx.TileShape(p.rows_per_rank(), p.local_cols()), fx.WRITE_ALLTOALL, True,
                     fx.default_opts(trace=1))
        comm.sync()
        ev = fx.comm.read_trace(comm, 0, p)
        path = tmp_path / "trace.json"
        fx.comm.write_chrome_trace(str(path), ev)
        d = json.loads(path.read_text())
        xs = d["traceEvents"]
        assert xs and all(x["ph"] == "X" and x["dur"] >= 0 for x in xs)
        ctas = [x for x in xs if x["name"].startswith("cta ")]
        assert len(ctas) >= 1 and all(x["tid"] >= 0 for x in ctas)
        kinds = {x["name"].split(" ")[0] for x in xs if x["tid"] == -1}
        assert {"tile_write", "reduce"} <= kinds
        n_events = sum(1 for e in ev if e["event"] != "launch")
        assert sum(1 for x in xs if x["tid"] == -1) == n_events
