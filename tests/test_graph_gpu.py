"""CUDA-graph capture and replay of the fused operators (flux_opts.graph_safe).

A graph-safe operator zeroes the flags / counters it uses before and after its
kernel, so a captured graph can be replayed on new inputs: every replay must
match the oracle on that replay's inputs, also when eager operators (which use
epoch-stamped flags and monotonic counters) run between replays."""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_2406_06858_b200 as fx  # noqa: E402
from paper_2406_06858_b200 import _native as N  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import gpu_harness as H  # noqa: E402

AG, RS = fx.ALLGATHER_GEMM, fx.GEMM_REDUCESCATTER


def _op(comm, p, opts, streams, push=False):
    tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
    if p.pattern == AG:
        comm.ag_gemm(p, tile, p.rows_per_rank(), fx.PUSH if push else fx.PULL, True, opts, streams)
    else:
        comm.gemm_rs(p, tile, fx.WRITE_ALLTOALL, True, opts, streams)


@pytest.mark.parametrize("case", [(AG, 256, 1024, 512, 4), (AG, 64, 2048, 1024, 8), (RS, 1024, 512, 512, 4),
                                  (RS, 4096, 4096, 512, 4), (RS, 40, 24, 72, 4), (RS, 512, 8192, 1024, 8),
                                  (AG, 1000, 600, 200, 2), (AG, 512, 1024, 256, 4, "push")],
                         ids=lambda c: "x".join(map(str, c)))
def test_graph_replay_matches_oracle(case):
    pat, m, n, k, tp = case[:5]
    push = len(case) > 5
    p = fx.ProblemSpec(m, n, k, tp, pat)
    side = torch.cuda.Stream()
    streams = [side.cuda_stream] * tp
    gopts = fx.default_opts(out_dtype=fx.F32, graph_safe=1, wall_budget_s=5.0)
    eopts = fx.default_opts(out_dtype=fx.F32, wall_budget_s=5.0)
    with H.make_comm(p) as comm:
        H.upload(comm, p, seed=1)
        with torch.cuda.stream(side):
            _op(comm, p, gopts, streams, push)  # warm-up: schedule tables are uploaded outside the capture
        comm.sync()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            _op(comm, p, gopts, streams, push)
        for it in range(4):
            a, b = H.upload(comm, p, seed=100 + it)
            if it == 2:  # an eager operator between replays (different inputs, normal epochs)
                _op(comm, p, eopts, None, push)
                comm.sync()
                a, b = H.upload(comm, p, seed=100 + it)
            graph.replay()
            torch.cuda.synchronize()
            want = O.dense_oracle(pat, m, n, k, tp, a, b)
            got = H.outputs(comm, p, True)
            for r in range(tp):
                assert O.max_rel_error(got[r], want[r]) <= H.tol(True, k), (it, r)
        # and eager operators still work after the replays
        a, b = H.upload(comm, p, seed=7)
        _op(comm, p, eopts, None)
        comm.sync()
        want = O.dense_oracle(pat, m, n, k, tp, a, b)
        got = H.outputs(comm, p, True)
        for r in range(tp):
            assert O.max_rel_error(got[r], want[r]) <= H.tol(True, k), ("eager", r)


def test_graph_replay_local_gemm_and_mlp():
    """The local GEMM (tail-split counters) and the chained MLP (AG-GEMM +
    SwiGLU -> GEMM-RS) captured and replayed."""
    tp, m, hidden, ffn = 4, 256, 512, 2048
    spec = fx.MlpSpec(m=m, hidden=hidden, ffn=ffn, tp=tp, activation=fx.ACT_SWIGLU)
    side = torch.cuda.Stream()
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    x = [torch.empty(m // tp, hidden, device="cuda", dtype=torch.bfloat16) for _ in range(tp)]
    f = ffn // tp  # SwiGLU: w_up holds 2f rows (128 gate + 128 up per 256-row group)
    wu = [(torch.randn(2 * f, hidden, device="cuda", generator=g) * 0.05).to(torch.bfloat16) for _ in range(tp)]
    wd = [(torch.randn(hidden, f, device="cuda", generator=g) * 0.05).to(torch.bfloat16) for _ in range(tp)]
    act = [torch.empty(m, f, device="cuda", dtype=torch.bfloat16) for _ in range(tp)]
    out = [torch.empty(m // tp, hidden, device="cuda", dtype=torch.bfloat16) for _ in range(tp)]
    ops = [dict(x=x[r], w_up=wu[r], w_down=wd[r], act=act[r], out=out[r]) for r in range(tp)]
    gopts = fx.default_opts(graph_safe=1)
    with fx.Communicator(tp, [0] * tp, heap_bytes=spec.required_heap_bytes()) as comm:
        for t in x:
            t.copy_(torch.randn(t.shape, device="cuda", generator=g).to(torch.bfloat16))
        with torch.cuda.stream(side):
            comm.mlp_forward(spec, ops, opts=gopts, streams=[side.cuda_stream] * tp)
        comm.sync()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            comm.mlp_forward(spec, ops, opts=gopts, streams=[side.cuda_stream] * tp)
        for it in range(3):
            for t in x:
                t.copy_(torch.randn(t.shape, device="cuda", generator=g).to(torch.bfloat16))
            torch.cuda.synchronize()
            graph.replay()
            torch.cuda.synchronize()
            xf = torch.cat([t.float() for t in x])
            for r in range(tp):
                h = xf @ wu[r].float().t()
                h = h.view(m, -1, 2, 128)
                a_r = (torch.nn.functional.silu(h[:, :, 0]) * h[:, :, 1]).reshape(m, -1)
                assert (act[r].float() - a_r).abs().max() <= 2e-2 * max(1.0, a_r.abs().max().item()), (it, r)
            full = sum(act[s].float() @ wd[s].float().t() for s in range(tp))
            for r in range(tp):
                ref = full[r * (m // tp):(r + 1) * (m // tp)]
                assert (out[r].float() - ref).abs().max() <= 3e-2 * max(1.0, ref.abs().max().item()), (it, r)

    p = fx.ProblemSpec(1000, 600, 2048, 1, AG)  # tail split on (ragged last wave, K long enough to split)
    with H.make_comm(p) as comm:
        st = [side.cuda_stream]
        gl = fx.default_opts(out_dtype=fx.F32, graph_safe=1)
        H.upload(comm, p, seed=5)
        with torch.cuda.stream(side):
            comm.local_gemm(p, gl, st)
        comm.sync()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            comm.local_gemm(p, gl, st)
        for it in range(3):
            a, b = H.upload(comm, p, seed=50 + it)
            comm.tensor(0, N.BUF_A_AGG, p).copy_(comm.tensor(0, N.BUF_A_SHARD, p))  # the local GEMM reads a_agg
            torch.cuda.synchronize()
            graph.replay()
            torch.cuda.synchronize()
            want = O.dense_oracle(AG, p.m, p.n, p.k, 1, a, b)
            got = H.outputs(comm, p, True)
            assert O.max_rel_error(got[0], want[0]) <= H.tol(True, p.k), it


def test_graph_safe_contract():
    """graph_safe is refused where it cannot hold: copy-engine AllGather,
    arrival-order FusedReduce, the unfused baseline."""
    p = fx.ProblemSpec(256, 512, 256, 2, AG)
    with H.make_comm(p) as comm:
        tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
        with pytest.raises(N.ConfigError, match="in-kernel transfer engine"):
            comm.ag_gemm(p, tile, p.rows_per_rank(), fx.PULL, True, fx.default_opts(graph_safe=1, ag_engine=1))
        with pytest.raises(N.ConfigError, match="fused operators"):
            comm.nonoverlap(p, fx.default_opts(graph_safe=1))
    q = fx.ProblemSpec(256, 512, 256, 2, RS)
    with H.make_comm(q) as comm:
        with pytest.raises(N.ConfigError, match="FusedReduce"):
            comm.gemm_rs(q, fx.TileShape(q.rows_per_rank(), q.local_cols()), fx.FUSED_REDUCE, True,
                         fx.default_opts(graph_safe=1, deterministic_reduce=0))
