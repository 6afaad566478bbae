"""The streaming decode kernel (flux_opts.decode_kernel, flux_stream_kernel):
weights on the MMA M side, tokens on N, stream-K over the weight shard with
K-segments summed in segment order. Checked against the CPU oracle at the
per-GPU decode shapes of BASELINE configs[4] (one GPU's share of Llama-2-70B
TP=8: tp=1 problems) and with ranks emulated on one GPU, through every mode
(local GEMM, AllGather-GEMM on both transfer engines, GEMM-ReduceScatter with
fp32 / bf16 partials), activations, graph replay, fault injection, and for
bit-identity across runs (the segment sum order is fixed)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_2406_06858_b200 as fx  # noqa: E402
from paper_2406_06858_b200 import _native as N  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import gpu_harness as H  # noqa: E402

AG, RS = fx.ALLGATHER_GEMM, fx.GEMM_REDUCESCATTER
STREAM = fx.DECODE_STREAM


def _run(comm, p, f32=True, **kw):
    kw.setdefault("wall_budget_s", 5.0)
    opts = fx.default_opts(out_dtype=fx.F32 if f32 else fx.BF16, **kw)
    tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
    if p.pattern == AG:
        comm.ag_gemm(p, tile, 0, fx.PULL, True, opts)
    else:
        comm.gemm_rs(p, tile, fx.WRITE_ALLTOALL, True, opts)
    comm.sync()
    return H.outputs(comm, p, f32)


# (pattern, m, n, k, tp): tp=1 rows are one GPU's share of configs[4] at TP=8
# (full K / N shard), small cases cover ragged n / k, odd token counts and
# K-segment counts from 1 to 8 per n-tile.
CASES = [(AG, 16, 3584, 8192, 1), (RS, 16, 8192, 3584, 1), (RS, 16, 8192, 1024, 1), (AG, 64, 3584, 8192, 1),
         (AG, 128, 1024, 2048, 1), (RS, 128, 2048, 1024, 1), (AG, 16, 1024, 512, 8), (RS, 16, 1024, 1024, 8),
         (RS, 64, 2048, 512, 4), (AG, 24, 600, 200, 2), (RS, 40, 24, 72, 4), (AG, 3, 130, 70, 1),
         (RS, 8, 136, 4096, 2), (AG, 100, 256, 64, 4),
         # one source per owner row (tp=1): the finish keeps four row groups per thread in flight
         (RS, 64, 8192, 1024, 1), (RS, 40, 200, 300, 1), (RS, 7, 136, 4096, 1),
         # cluster ring mode with each CTA summing its own 16-row chunks (compact slots)
         (AG, 128, 3584, 8192, 1), (AG, 48, 3584, 4096, 1), (AG, 100, 1024, 2048, 1)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c)))
def test_stream_kernel_matches_oracle(case):
    pat, m, n, k, tp = case
    p = fx.ProblemSpec(m, n, k, tp, pat)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=11)
        want = O.dense_oracle(pat, m, n, k, tp, a, b)
        for f32 in (True, False):
            got = _run(comm, p, f32, decode_kernel=STREAM)
            for r in range(tp):
                assert O.max_rel_error(got[r], want[r]) <= H.tol(f32, k), (f32, r)


@pytest.mark.parametrize("case", [(AG, 16, 3584, 8192, 1), (RS, 16, 8192, 3584, 1), (RS, 48, 4096, 2048, 4)],
                         ids=lambda c: "x".join(map(str, c)))
def test_stream_kernel_bit_identical_across_runs(case):
    """Split n-tiles are summed in K-segment order by fixed CTAs, whichever
    segment lands last: repeated runs give identical bits."""
    pat, m, n, k, tp = case
    p = fx.ProblemSpec(m, n, k, tp, pat)
    with H.make_comm(p) as comm:
        H.upload(comm, p, seed=5)
        first = _run(comm, p, True, decode_kernel=STREAM)
        for seed in (0, 3):
            again = _run(comm, p, True, decode_kernel=STREAM, interleave_seed=seed)
            for r in range(tp):
                assert np.array_equal(first[r], again[r]), (seed, r)


@pytest.mark.parametrize("case,auto_kernel", [((AG, 16, 3584, 8192), STREAM), ((RS, 128, 8192, 1024), STREAM),
                                               ((AG, 128, 1024, 2048), STREAM), ((AG, 256, 1024, 2048), fx.DECODE_TILE)],
                         ids=["ag16-stream", "rs128-stream", "ag128-stream", "ag256-tile"])
def test_stream_kernel_is_the_auto_choice_for_one_rank_per_gpu_decode(case, auto_kernel):
    """Auto (decode_kernel=0) with one rank per GPU takes the streaming kernel
    up to 128 rows and the tile kernel above: outputs bit-identical to the
    forced choice; both kernels within tolerance of the oracle (their K orders
    differ)."""
    pat, m, n, k = case
    p = fx.ProblemSpec(m, n, k, 1, pat)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=2)
        auto = _run(comm, p, True)
        forced = _run(comm, p, True, decode_kernel=auto_kernel)
        other = _run(comm, p, True, decode_kernel=fx.DECODE_TILE if auto_kernel == STREAM else STREAM)
        assert np.array_equal(auto[0], forced[0])
        want = O.dense_oracle(pat, m, n, k, 1, a, b)
        assert O.max_rel_error(auto[0], want[0]) <= H.tol(True, k)
        assert O.max_rel_error(other[0], want[0]) <= H.tol(True, k)


@pytest.mark.parametrize("engine", [1, 2])
def test_stream_kernel_allgather_engines(engine):
    """Gathered token rows from the copy-engine transfer loop (comm-tile flags)
    or the in-kernel transfer (piece counters), ranks emulated on one GPU."""
    p = fx.ProblemSpec(32, 2048, 1024, 8, AG)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=4)
        want = O.dense_oracle(AG, p.m, p.n, p.k, p.tp, a, b)
        got = _run(comm, p, True, decode_kernel=STREAM, ag_engine=engine)
        for r in range(p.tp):
            assert O.max_rel_error(got[r], want[r]) <= H.tol(True, p.k), r


def test_stream_kernel_rs_bf16_partials():
    p = fx.ProblemSpec(32, 4096, 2048, 4, RS)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=8)
        want = O.dense_oracle(RS, p.m, p.n, p.k, p.tp, a, b)
        got = _run(comm, p, True, decode_kernel=STREAM, rs_partials=fx.BF16)
        for r in range(p.tp):
            assert O.normwise_error(got[r], want[r]) <= 5e-3, r


@pytest.mark.parametrize("act", [fx.ACT_GELU, fx.ACT_RELU, fx.ACT_SILU])
def test_stream_kernel_epilogue_activation(act):
    """AG-GEMM + activation on the streaming kernel against a torch fp32
    reference of the same bf16 operands (the oracle has no activations)."""
    p = fx.ProblemSpec(16, 1024, 2048, 2, AG)
    fn = {fx.ACT_GELU: torch.nn.functional.gelu, fx.ACT_RELU: torch.relu, fx.ACT_SILU: torch.nn.functional.silu}[act]
    with H.make_comm(p) as comm:
        H.upload(comm, p, seed=9)
        got = _run(comm, p, True, decode_kernel=STREAM, activation=act)
        a = torch.cat([comm.tensor(r, N.BUF_A_SHARD, p).float() for r in range(p.tp)])
        for r in range(p.tp):
            want = fn(a @ comm.tensor(r, N.BUF_B_SHARD, p).float().t()).double().cpu().numpy()
            assert O.max_rel_error(got[r], want) <= 1e-3, r


def test_stream_kernel_local_gemm_matches_torch():
    p = fx.ProblemSpec(16, 3584, 8192, 1, AG)
    with H.make_comm(p) as comm:
        H.upload(comm, p, seed=6)
        # the local GEMM of the AllGather pattern reads the gathered buffer: fill it
        _run(comm, p, True, decode_kernel=STREAM)
        comm.local_gemm(p, fx.default_opts(out_dtype=fx.F32, decode_kernel=STREAM))
        comm.sync()
        got = comm.tensor(0, N.BUF_C_OUT_F32, p).double().cpu().numpy()
        a = comm.tensor(0, N.BUF_A_SHARD, p).float()
        want = (a @ comm.tensor(0, N.BUF_B_SHARD, p).float().t()).double().cpu().numpy()
        assert O.max_rel_error(got, want) <= H.tol(True, p.k)


@pytest.mark.parametrize("case", [(AG, 16, 3584, 8192, 1), (RS, 16, 8192, 3584, 1), (RS, 32, 2048, 1024, 4)],
                         ids=lambda c: "x".join(map(str, c)))
def test_stream_kernel_graph_replay(case):
    """Graph-safe streaming operators: the segment flags carry a per-launch tag
    that a replay repeats, so the operator zeroes them before its kernel."""
    pat, m, n, k, tp = case
    p = fx.ProblemSpec(m, n, k, tp, pat)
    side = torch.cuda.Stream()
    streams = [side.cuda_stream] * tp
    gopts = fx.default_opts(out_dtype=fx.F32, graph_safe=1, wall_budget_s=5.0, decode_kernel=STREAM)
    tile = fx.TileShape(p.rows_per_rank(), p.local_cols())

    def op(opts, st):
        if pat == AG:
            comm.ag_gemm(p, tile, p.rows_per_rank(), fx.PULL, True, opts, st)
        else:
            comm.gemm_rs(p, tile, fx.WRITE_ALLTOALL, True, opts, st)

    with H.make_comm(p) as comm:
        H.upload(comm, p, seed=1)
        with torch.cuda.stream(side):
            op(gopts, streams)
        comm.sync()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            op(gopts, streams)
        for it in range(3):
            a, b = H.upload(comm, p, seed=200 + it)
            if it == 1:
                op(fx.default_opts(out_dtype=fx.F32, decode_kernel=STREAM), None)
                comm.sync()
            graph.replay()
            torch.cuda.synchronize()
            want = O.dense_oracle(pat, m, n, k, tp, a, b)
            got = H.outputs(comm, p, True)
            for r in range(tp):
                assert O.max_rel_error(got[r], want[r]) <= H.tol(True, k), (it, r)


def test_stream_kernel_dropped_rs_flag_raises_deadlock_error():
    """A dropped (n-tile, source) flag leaves the owner's epilogue waiting for
    that source's partial: the bounded device wait raises DeadlockError naming
    the flag, and the communicator runs the next operator correctly."""
    p = fx.ProblemSpec(16, 1024, 512, 2, RS)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=3)
        comm.inject_fault(fx.FAULT_DROP_SIGNAL, 1, 2)  # owner 1, flag (n-tile 1) x tp 2 + source 0
        with pytest.raises(fx.DeadlockError) as ei:
            _run(comm, p, True, decode_kernel=STREAM, wall_budget_s=0.5)
        assert "waiting for partial of tile 1 from source 0" in str(ei.value), str(ei.value)
        got = _run(comm, p, True, decode_kernel=STREAM)
        want = O.dense_oracle(RS, p.m, p.n, p.k, p.tp, a, b)
        for r in range(p.tp):
            assert O.max_rel_error(got[r], want[r]) <= H.tol(True, p.k), r


def test_stream_kernel_rs_many_ranks_per_launch_stays_deadlock_free():
    """Several emulated ranks in one launch with more n-tiles than SMs: a
    streaming GEMM-RS would wait on tiles ahead of its own range (the slot
    wrap), so the request runs on the tile kernel and stays right."""
    p = fx.ProblemSpec(16, 8192, 3584, 8, RS)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=21)
        got = _run(comm, p, True, decode_kernel=STREAM, wall_budget_s=5.0)
        rows = [[0, 1]] * 8
        for r in range(8):
            want = O.rs_rows(p.m, p.n, p.k, 8, a, b, r, rows[r])
            assert O.max_rel_error(got[r][rows[r]], want) <= H.tol(True, p.k), r

