"""Chained tensor-parallel MLP (paper Fig. 2): epilogue
activations of the AllGather-GEMM, the AG-GEMM -> GEMM-RS forward chain and the
backward-of-input interchange, against a plain PyTorch fp32 reference on the
same bf16 inputs (the oracle for these floating-point epilogues).

Tolerance: bf16 operands, fp32 accumulation, bf16 intermediates and outputs;
max |got - ref| / max(1, max |ref|) <= 1.5e-2 (two bf16 roundings, 2^-8 each,
plus the activation's fp32 evaluation)."""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_2406_06858_b200 as fx  # noqa: E402
from paper_2406_06858_b200 import _native as N  # noqa: E402

TOL = 1.5e-2
ACTS = {fx.ACT_GELU: lambda y: torch.nn.functional.gelu(y), fx.ACT_RELU: torch.relu,
        fx.ACT_SILU: torch.nn.functional.silu}


def _err(got, ref):
    got, ref = got.float(), ref.float()
    return ((got - ref).abs().max() / max(1.0, ref.abs().max().item())).item()


def _bf(shape, g, scale=1.0):
    return (torch.rand(shape, generator=g, device="cuda") * 2 - 1).mul_(scale).to(torch.bfloat16)


def _ag_case(tp, m, n, k, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    shards = [_bf((m // tp, k), g) for _ in range(tp)]
    weights = [_bf((n // tp, k), g, 0.1) for _ in range(tp)]
    return shards, weights, torch.cat(shards).float()


@pytest.mark.parametrize("act", [fx.ACT_GELU, fx.ACT_RELU, fx.ACT_SILU])
@pytest.mark.parametrize("engine", [1, 2])
def test_ag_gemm_activation_epilogue(act, engine):
    tp, m, n, k = 4, 512, 1024, 384
    p = fx.ProblemSpec(m, n, k, tp, fx.ALLGATHER_GEMM)
    shards, weights, x = _ag_case(tp, m, n, k, 11 + act)
    outs = [torch.empty(m, n // tp, dtype=torch.bfloat16, device="cuda") for _ in range(tp)]
    pres = [torch.empty(m, n // tp, dtype=torch.bfloat16, device="cuda") for _ in range(tp)]
    with fx.Communicator(tp, [0] * tp, heap_bytes=fx.required_heap_bytes(p)) as comm:
        opts = fx.default_opts(activation=act, ag_engine=engine, wall_budget_s=5.0)
        comm.ag_gemm_ex(p, fx.TileShape(m // tp, n // tp), list(zip(shards, weights, outs, pres)), opts=opts)
        comm.sync()
    for r in range(tp):
        y = x @ weights[r].float().t()
        assert _err(pres[r], y) <= TOL, ("pre", r)
        assert _err(outs[r], ACTS[act](y)) <= TOL, ("act", r)


def test_ag_gemm_swiglu_epilogue():
    tp, m, n, k = 2, 256, 1024, 256  # local n = 512: two groups of 128 gate + 128 up columns
    p = fx.ProblemSpec(m, n, k, tp, fx.ALLGATHER_GEMM)
    shards, weights, x = _ag_case(tp, m, n, k, 5)
    outs = [torch.empty(m, n // tp // 2, dtype=torch.bfloat16, device="cuda") for _ in range(tp)]
    with fx.Communicator(tp, [0] * tp, heap_bytes=fx.required_heap_bytes(p)) as comm:
        comm.ag_gemm_ex(p, fx.TileShape(m // tp, n // tp), [(a, b, c) for a, b, c in zip(shards, weights, outs)],
                        opts=fx.default_opts(activation=fx.ACT_SWIGLU, wall_budget_s=5.0))
        comm.sync()
    for r in range(tp):
        y = (x @ weights[r].float().t()).view(m, -1, 2, 128)
        ref = (torch.nn.functional.silu(y[:, :, 0]) * y[:, :, 1]).reshape(m, -1)
        assert _err(outs[r], ref) <= TOL, r


def test_activation_contract_errors():
    tp, m, n, k = 2, 256, 768, 128
    p = fx.ProblemSpec(m, n, k, tp, fx.ALLGATHER_GEMM)
    with fx.Communicator(tp, [0] * tp, heap_bytes=64 << 20) as comm:
        t = fx.TileShape(m // tp, n // tp)
        with pytest.raises(fx.ShapeError):  # local n = 384 is not a multiple of 256
            comm.ag_gemm(p, t, opts=fx.default_opts(activation=fx.ACT_SWIGLU))
        with pytest.raises(fx.ConfigError):  # derivative without the saved pre-activation
            comm.ag_gemm(p, t, opts=fx.default_opts(activation_grad=fx.ACT_GELU))
        prs = fx.ProblemSpec(m, 256, 256, tp, fx.GEMM_REDUCESCATTER)
        with pytest.raises(fx.ConfigError):  # activations belong to the AG-GEMM
            comm.gemm_rs(prs, fx.TileShape(m // tp, 256), opts=fx.default_opts(activation=fx.ACT_GELU))


def _mlp_inputs(spec, seed, swiglu=False):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    tp, f = spec.tp, spec.ffn // spec.tp
    x = [_bf((spec.m // tp, spec.hidden), g) for _ in range(tp)]
    w_up = [_bf((f * (2 if swiglu else 1), spec.hidden), g, 0.1) for _ in range(tp)]
    w_down = [_bf((spec.hidden, f), g, 0.1) for _ in range(tp)]
    return x, w_up, w_down


@pytest.mark.parametrize("act,m", [(fx.ACT_GELU, 1024), (fx.ACT_SILU, 1024), (fx.ACT_SWIGLU, 1024),
                                   (fx.ACT_SWIGLU, 64), (fx.ACT_GELU, 40)])
def test_mlp_forward_chain(act, m):
    """m = 64 / 40: decode-sized ownership blocks (owner-unit GEMM-RS into the
    caller's output)."""
    spec = fx.MlpSpec(m=m, hidden=512, ffn=2048, tp=4, activation=act)
    tp, f = spec.tp, spec.ffn // spec.tp
    x, w_up, w_down = _mlp_inputs(spec, 21 + act, swiglu=act == fx.ACT_SWIGLU)
    inter = [torch.empty(spec.m, f, dtype=torch.bfloat16, device="cuda") for _ in range(tp)]
    out = [torch.empty(spec.m // tp, spec.hidden, dtype=torch.bfloat16, device="cuda") for _ in range(tp)]
    with fx.Communicator(tp, [0] * tp, heap_bytes=spec.required_heap_bytes()) as comm:
        comm.mlp_forward(spec, [dict(x=x[r], w_up=w_up[r], w_down=w_down[r], act=inter[r], out=out[r])
                                for r in range(tp)], opts=fx.default_opts(wall_budget_s=5.0))
        comm.sync()
    xa = torch.cat(x).float()
    total = torch.zeros(spec.m, spec.hidden, device="cuda")
    for r in range(tp):
        y = xa @ w_up[r].float().t()
        if act == fx.ACT_SWIGLU:
            y4 = y.view(spec.m, -1, 2, 128)
            a = (torch.nn.functional.silu(y4[:, :, 0]) * y4[:, :, 1]).reshape(spec.m, -1)
        else:
            a = ACTS[act](y)
        assert _err(inter[r], a) <= TOL, ("intermediate", r)
        total += a.to(torch.bfloat16).float() @ w_down[r].float().t()
    rpr = spec.m // tp
    for r in range(tp):
        assert _err(out[r], total[r * rpr:(r + 1) * rpr]) <= TOL, ("out", r)


def _swiglu_ref(y):
    y4 = y.view(y.shape[0], -1, 2, 128)
    return (torch.nn.functional.silu(y4[:, :, 0]) * y4[:, :, 1]).reshape(y.shape[0], -1)


@pytest.mark.parametrize("act", [fx.ACT_GELU, fx.ACT_RELU, fx.ACT_SILU, fx.ACT_SWIGLU])
def test_mlp_backward_dx_matches_autograd(act):
    """dx of the TP MLP: AG-GEMM(dout, W_down) * act'(pre) -> GEMM-RS with W_up
    (the AG <-> RS interchange of the backward pass); SWIGLU:
    dgate / dup from the saved gate / up pre-activations."""
    spec = fx.MlpSpec(m=512, hidden=256, ffn=1024, tp=2, activation=act)
    tp, f, rpr = spec.tp, spec.ffn // spec.tp, spec.m // spec.tp
    glu = act == fx.ACT_SWIGLU
    x, w_up, w_down = _mlp_inputs(spec, 7 + act, swiglu=glu)
    g = torch.Generator(device="cuda")
    g.manual_seed(99)
    dout = [_bf((rpr, spec.hidden), g) for _ in range(tp)]
    wide = 2 * f if glu else f
    pre = [torch.empty(spec.m, wide, dtype=torch.bfloat16, device="cuda") for _ in range(tp)]
    inter = [torch.empty(spec.m, f, dtype=torch.bfloat16, device="cuda") for _ in range(tp)]
    out = [torch.empty(rpr, spec.hidden, dtype=torch.bfloat16, device="cuda") for _ in range(tp)]
    dact = [torch.empty(spec.m, wide, dtype=torch.bfloat16, device="cuda") for _ in range(tp)]
    dx = [torch.empty(rpr, spec.hidden, dtype=torch.bfloat16, device="cuda") for _ in range(tp)]
    with fx.Communicator(tp, [0] * tp, heap_bytes=spec.required_heap_bytes()) as comm:
        opts = fx.default_opts(wall_budget_s=5.0)
        comm.mlp_forward(spec, [dict(x=x[r], w_up=w_up[r], w_down=w_down[r], pre=pre[r], act=inter[r], out=out[r])
                                for r in range(tp)], opts=opts)
        comm.mlp_backward_dx(spec, [dict(dout=dout[r], w_down_t=w_down[r].t().contiguous(),
                                         w_up_t=w_up[r].t().contiguous(), pre=pre[r], dact=dact[r], dx=dx[r])
                                    for r in range(tp)], opts=opts)
        comm.sync()
    # fp32 autograd reference of the same TP MLP on the same bf16 inputs
    xa = torch.cat(x).float().requires_grad_(True)
    fn = _swiglu_ref if glu else ACTS[act]
    y = sum(fn(xa @ w_up[r].float().t()) @ w_down[r].float().t() for r in range(tp))
    y.backward(torch.cat(dout).float())
    for r in range(tp):
        assert _err(dx[r], xa.grad[r * rpr:(r + 1) * rpr]) <= 2 * TOL, r
