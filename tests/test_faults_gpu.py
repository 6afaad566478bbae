"""Fault injection on the device paths (the reference's deadlock and double-set
checks): a dropped signal makes the waiting tile time out, the operator's
failure names the flag (spin_wait, engine.cpp:149-162; acceptance.cpp:121-158
catches DeadlockError), the next operator call reports it without a host
synchronisation, flux_sync clears it, and the communicator then runs clean and
matches the oracle again. A flag raised twice is an error when the detector
is on (SignalBoard::set, signal_board.hpp:25-28; engine.cpp:401-403).
"""
import re

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_2406_06858_b200 as fx  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import gpu_harness as H  # noqa: E402

AG, RS = fx.ALLGATHER_GEMM, fx.GEMM_REDUCESCATTER
BUDGET = 0.3  # seconds: the injected fault's waiter times out after this


def _op(comm, p, engine=0, rpct=0, **kw):
    opts = fx.default_opts(out_dtype=fx.F32, wall_budget_s=BUDGET, ag_engine=engine, **kw)
    if p.pattern == AG:
        comm.ag_gemm(p, fx.TileShape(p.rows_per_rank(), p.local_cols()), rpct or p.rows_per_rank(), fx.PULL, True,
                     opts)
    else:
        comm.gemm_rs(p, fx.TileShape(p.rows_per_rank(), p.local_cols()), fx.WRITE_ALLTOALL, True, opts)


def _clean_run_matches(comm, p, a, b, **kw):
    _op(comm, p, **kw)
    comm.sync()
    want = O.dense_oracle(p.pattern, p.m, p.n, p.k, p.tp, a, b)
    got = H.outputs(comm, p, True)
    for r in range(p.tp):
        assert O.max_rel_error(got[r], want[r]) <= H.tol(True, p.k), r


def _rs_flag(p, owner, src, tn=0):
    """Index of RS flag (tile, src) for the first 128-row tile of owner's block."""
    tiles_n = (p.n + 255) // 256
    tile = (owner * p.rows_per_rank() // 128) * tiles_n + tn
    return tile * p.tp + src, tile


@pytest.mark.parametrize("engine", [1, 2], ids=["copy_engine", "in_kernel"])
def test_dropped_allgather_signal_raises_deadlock(engine):
    p = fx.ProblemSpec(512, 512, 256, 4, AG)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=5)
        rank = 2
        # copy engines: comm tile 1 (rows 128..255) of rank 2's board (rpct = 128);
        # in-kernel: 128-row group 1 of rank 2's a_agg
        comm.inject_fault(fx.FAULT_DROP_SIGNAL, rank, 1)
        _op(comm, p, engine=engine, rpct=128)
        torch.cuda.synchronize()
        # The next operator reports the failure without synchronising ...
        with pytest.raises(fx.DeadlockError, match="previous operator failed"):
            _op(comm, p, engine=engine, rpct=128)
        # ... flux_sync names the flag (reference spin_wait text) and clears it.
        with pytest.raises(fx.DeadlockError) as ei:
            comm.sync()
        msg = str(ei.value)
        assert re.search(r"deadlock budget exhausted waiting for signal 1 for tile \(\d+,\d+\) on rank 2", msg), msg
        comm.sync()  # cleared
        _clean_run_matches(comm, p, a, b, engine=engine, rpct=128)


@pytest.mark.parametrize("case", [(RS, 2048, 2048, 64, 4), (RS, 64, 512, 256, 4), (RS, 2048, 4864, 64, 4),
                                  (RS, 1024, 512, 256, 4)],
                         ids=["owner_sum", "decode_units", "chain", "subwave_units"])
def test_dropped_reducescatter_signal_raises_deadlock(case):
    pat, m, n, k, tp = case
    p = fx.ProblemSpec(m, n, k, tp, pat)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=6)
        owner, src = 1, 0
        idx, tile = _rs_flag(p, owner, src)
        comm.inject_fault(fx.FAULT_DROP_SIGNAL, owner, idx)
        _op(comm, p)
        with pytest.raises(fx.DeadlockError) as ei:
            comm.sync()
        msg = str(ei.value)
        assert f"deadlock budget exhausted waiting for partial of tile {tile} from source" in msg, msg
        _clean_run_matches(comm, p, a, b)


def test_fault_is_armed_for_one_operator_only():
    p = fx.ProblemSpec(512, 512, 256, 2, RS)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=8)
        idx, _ = _rs_flag(p, 1, 0)
        comm.inject_fault(fx.FAULT_DROP_SIGNAL, 1, idx)
        _op(comm, p)
        with pytest.raises(fx.DeadlockError):
            comm.sync()
        _clean_run_matches(comm, p, a, b)
        _clean_run_matches(comm, p, a, b)


def test_double_set_reducescatter_flag_detected():
    p = fx.ProblemSpec(1024, 512, 256, 4, RS)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=9)
        idx, _ = _rs_flag(p, 2, 3)
        # Detector off: a doubled stamp is idempotent, the result is still right.
        comm.inject_fault(fx.FAULT_DOUBLE_SIGNAL, 2, idx)
        _clean_run_matches(comm, p, a, b)
        # Detector on: the second stamp is an error naming the flag.
        comm.set_check_double_set(True)
        comm.inject_fault(fx.FAULT_DOUBLE_SIGNAL, 2, idx)
        _op(comm, p)
        with pytest.raises(fx.SignalError, match=f"flag {idx} on rank 2 set twice"):
            comm.sync()
        _clean_run_matches(comm, p, a, b)  # detector on, no fault: clean
        comm.set_check_double_set(False)


def test_double_set_copy_engine_flag_detected_on_host():
    p = fx.ProblemSpec(512, 512, 256, 4, AG)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=10)
        comm.inject_fault(fx.FAULT_DOUBLE_SIGNAL, 3, 0)
        with pytest.raises(fx.SignalError, match="flag 0 on rank 3 set twice"):
            _op(comm, p, engine=1, rpct=64)
        comm.sync()  # everything was enqueued: the device work completes normally
        _clean_run_matches(comm, p, a, b, engine=1, rpct=64)


def test_pending_failure_surfaces_through_torch_op():
    """The PyTorch custom ops never call flux_sync: a device failure left by an
    earlier operator must still make the next op call raise instead of
    silently computing on stale signals (sticky error word)."""
    from paper_2406_06858_b200 import torch_ops as T

    p = fx.ProblemSpec(512, 512, 256, 2, RS)
    with H.make_comm(p) as comm:
        H.upload(comm, p, seed=11)
        idx, _ = _rs_flag(p, 1, 0)
        comm.inject_fault(fx.FAULT_DROP_SIGNAL, 1, idx)
        _op(comm, p)
        torch.cuda.synchronize()
        cid = T.register(comm)
        x = torch.zeros(p.rows_per_rank(), 256, dtype=torch.bfloat16, device="cuda")
        w = torch.zeros(256, 256, dtype=torch.bfloat16, device="cuda")
        with pytest.raises(fx.DeadlockError, match="previous operator failed"):
            torch.ops.flux_b200.ag_gemm(x, w, cid)
        with pytest.raises(fx.DeadlockError):
            comm.sync()
        T._REGISTRY.pop(cid, None)


def test_torch_op_operand_validation():
    from paper_2406_06858_b200 import torch_ops as T

    p = fx.ProblemSpec(512, 512, 256, 2, AG)
    with H.make_comm(p) as comm:
        cid = T.register(comm)
        x = torch.zeros(256, 256, dtype=torch.bfloat16, device="cuda")
        with pytest.raises(ValueError, match="bfloat16"):
            torch.ops.flux_b200.ag_gemm(x.float(), torch.zeros(256, 256, dtype=torch.bfloat16, device="cuda"), cid)
        with pytest.raises(ValueError, match="columns"):
            torch.ops.flux_b200.ag_gemm(x, torch.zeros(256, 128, dtype=torch.bfloat16, device="cuda"), cid)
        with pytest.raises(ValueError, match="row-major"):
            torch.ops.flux_b200.ag_gemm(x.t(), torch.zeros(256, 256, dtype=torch.bfloat16, device="cuda"), cid)
        T._REGISTRY.pop(cid, None)
