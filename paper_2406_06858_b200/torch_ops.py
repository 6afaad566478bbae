"""PyTorch custom ops over the fused operators: the paper's
integration point, where Megatron/vLLM MLP blocks call AG-GEMM / GEMM-RS on
torch tensors. One process per GPU; the communicator is created
once (IPC handles exchanged through torch.distributed) and registered here.

    comm_id = torch_ops.init_process_group_communicator(max_problem)
    out = torch.ops.flux_b200.ag_gemm(x_shard, w_shard, comm_id)   # [m, n/tp]
    y   = torch.ops.flux_b200.gemm_rs(h_local, w2_shard, comm_id)  # [m/tp, n]
"""
from __future__ import annotations

import itertools

import torch

from . import _native as N
from .comm import Communicator, ProblemSpec, TileShape, required_heap_bytes

_REGISTRY: dict[int, Communicator] = {}
_IDS = itertools.count(1)


def register(comm: Communicator) -> int:
    cid = next(_IDS)
    _REGISTRY[cid] = comm
    return cid


def init_process_group_communicator(max_problem: ProblemSpec, group=None) -> int:
    """IPC communicator over the default torch.distributed group, sized for the
    largest problem it will run; returns the id the ops take."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)

    def gather(blob):
        out = [None] * world
        dist.all_gather_object(out, blob, group=group)
        return out

    comm = Communicator.ipc(rank, world, torch.cuda.current_device(), required_heap_bytes(max_problem) + (8 << 20),
                            gather)
    return register(comm)


def _check_mat(name: str, t: torch.Tensor, comm: Communicator, rows: int | None = None,
               cols: int | None = None) -> None:
    """The C ABI carries only (pointer, row pitch): everything else about a
    caller tensor is checked here, before the kernels build TMA maps over it."""
    if not isinstance(t, torch.Tensor) or t.dim() != 2:
        raise ValueError(f"{name}: expected a 2-D tensor")
    if t.dtype != torch.bfloat16:
        raise ValueError(f"{name}: expected bfloat16, got {t.dtype}")
    if not t.is_cuda:
        raise ValueError(f"{name}: expected a CUDA tensor")
    dev = getattr(comm, "device", None)
    if dev is not None and t.device.index != dev:
        raise ValueError(f"{name}: on cuda:{t.device.index}, the communicator runs on cuda:{dev}")
    if t.shape[0] > 1 and (t.stride(1) != 1 or t.stride(0) < t.shape[1]):
        raise ValueError(f"{name}: expected a row-major view (stride(1) == 1, stride(0) >= cols), "
                         f"got strides {tuple(t.stride())} for shape {tuple(t.shape)}")
    if t.shape[0] <= 1 and t.stride(1) != 1:
        raise ValueError(f"{name}: expected unit column stride")
    if t.data_ptr() % 16 or (t.stride(0) * 2) % 16:
        raise ValueError(f"{name}: base address and row pitch must be 16-byte aligned (TMA)")
    if rows is not None and t.shape[0] != rows:
        raise ValueError(f"{name}: expected {rows} rows, got {t.shape[0]}")
    if cols is not None and t.shape[1] != cols:
        raise ValueError(f"{name}: expected {cols} columns, got {t.shape[1]}")


def _stream():
    """torch's current stream as a cudaStream_t. torch reports the legacy
    default stream as 0, which the C ABI reads as "library stream": pass
    cudaStreamLegacy (0x1) instead so the op is ordered with torch's work."""
    s = torch.cuda.current_stream().cuda_stream
    return [s if s != 0 else 1]


@torch.library.custom_op("flux_b200::ag_gemm", mutates_args=())
def ag_gemm(a_shard: torch.Tensor, weight: torch.Tensor, comm_id: int) -> torch.Tensor:
    """AllGather(a_shard) @ weight^T. a_shard [m/tp, k] bf16, weight [n/tp, k]
    bf16 (nn.Linear layout); returns [m, n/tp] bf16."""
    comm = _REGISTRY[comm_id]
    tp, k = comm.tp, a_shard.shape[1]
    _check_mat("a_shard", a_shard, comm)
    _check_mat("weight", weight, comm, cols=k)
    p = ProblemSpec(a_shard.shape[0] * tp, weight.shape[0] * tp, k, tp, N.ALLGATHER_GEMM)
    out = torch.empty(p.m, weight.shape[0], dtype=torch.bfloat16, device=a_shard.device)
    comm.ag_gemm_ex(p, TileShape(p.rows_per_rank(), p.local_cols()), [(a_shard, weight, out)], streams=_stream())
    return out


@ag_gemm.register_fake
def _(a_shard, weight, comm_id):
    return a_shard.new_empty(a_shard.shape[0] * _REGISTRY[comm_id].tp, weight.shape[0])


@torch.library.custom_op("flux_b200::gemm_rs", mutates_args=())
def gemm_rs(a: torch.Tensor, weight: torch.Tensor, comm_id: int, b_kn: bool = False) -> torch.Tensor:
    """ReduceScatter(a @ weight^T) over rows. a [m, k/tp] bf16, weight [n, k/tp]
    bf16 (b_kn: weight given as [k/tp, n], used as a @ weight); returns this
    rank's [m/tp, n] bf16 rows (fixed-order fp32 sum)."""
    comm = _REGISTRY[comm_id]
    tp = comm.tp
    _check_mat("a", a, comm)
    if b_kn:
        _check_mat("weight", weight, comm, rows=a.shape[1])
    else:
        _check_mat("weight", weight, comm, cols=a.shape[1])
    n = weight.shape[1] if b_kn else weight.shape[0]
    p = ProblemSpec(a.shape[0], n, a.shape[1] * tp, tp, N.GEMM_REDUCESCATTER)
    out = torch.empty(p.rows_per_rank(), p.n, dtype=torch.bfloat16, device=a.device)
    comm.gemm_rs_ex(p, TileShape(p.rows_per_rank(), p.local_cols()), [(a, weight, out)],
                    opts=N.default_opts(b_layout=N.B_KN if b_kn else N.B_NK), streams=_stream())
    return out


@gemm_rs.register_fake
def _(a, weight, comm_id, b_kn=False):
    return a.new_empty(a.shape[0] // _REGISTRY[comm_id].tp, weight.shape[1] if b_kn else weight.shape[0])


# ---------------------------------------------------------------------------
# Chained tensor-parallel MLP as custom ops + autograd.
# ---------------------------------------------------------------------------
def _ag_problem(comm, a_shard, n_local):
    tp = comm.tp
    return ProblemSpec(a_shard.shape[0] * tp, n_local * tp, a_shard.shape[1], tp, N.ALLGATHER_GEMM)


@torch.library.custom_op("flux_b200::ag_gemm_act", mutates_args=())
def ag_gemm_act(a_shard: torch.Tensor, weight: torch.Tensor, comm_id: int,
                activation: int) -> tuple[torch.Tensor, torch.Tensor]:
    """activation(AllGather(a_shard) @ weight^T) with the activation in the
    GEMM epilogue; also returns the pre-activation [m, n/tp] (SWIGLU: the output
    has half the columns — 128 gate + 128 up rows per 256-row weight group)."""
    comm = _REGISTRY[comm_id]
    _check_mat("a_shard", a_shard, comm)
    _check_mat("weight", weight, comm, cols=a_shard.shape[1])
    p = _ag_problem(comm, a_shard, weight.shape[0])
    swiglu = activation == N.ACT_SWIGLU
    out = torch.empty(p.m, weight.shape[0] // (2 if swiglu else 1), dtype=torch.bfloat16, device=a_shard.device)
    pre = torch.empty(p.m, weight.shape[0], dtype=torch.bfloat16, device=a_shard.device)
    opts = N.default_opts(activation=activation)
    comm.ag_gemm_ex(p, TileShape(p.rows_per_rank(), p.local_cols()), [(a_shard, weight, out, pre)],
                    opts=opts, streams=_stream())
    return out, pre


@ag_gemm_act.register_fake
def _(a_shard, weight, comm_id, activation):
    m = a_shard.shape[0] * _REGISTRY[comm_id].tp
    swiglu = activation == N.ACT_SWIGLU
    return a_shard.new_empty(m, weight.shape[0] // (2 if swiglu else 1)), a_shard.new_empty(m, weight.shape[0])


@torch.library.custom_op("flux_b200::ag_gemm_dact", mutates_args=())
def ag_gemm_dact(a_shard: torch.Tensor, weight: torch.Tensor, pre: torch.Tensor, comm_id: int,
                 activation: int, b_kn: bool = False) -> torch.Tensor:
    """(AllGather(a_shard) @ weight^T) * activation'(pre): the backward of the
    GEMM-RS + activation, with the derivative in the AG-GEMM epilogue (SWIGLU:
    dgate / dup in the gate/up grouping, twice the columns). b_kn: weight given
    as [k, n/tp] (e.g. the forward's W_down itself), used as AllGather(a) @ weight."""
    comm = _REGISTRY[comm_id]
    _check_mat("a_shard", a_shard, comm)
    if b_kn:
        _check_mat("weight", weight, comm, rows=a_shard.shape[1])
    else:
        _check_mat("weight", weight, comm, cols=a_shard.shape[1])
    n_local = weight.shape[1] if b_kn else weight.shape[0]
    p = _ag_problem(comm, a_shard, n_local)
    width = n_local * (2 if activation == N.ACT_SWIGLU else 1)
    _check_mat("pre", pre, comm, rows=p.m, cols=width)
    out = torch.empty(p.m, width, dtype=torch.bfloat16, device=a_shard.device)
    comm.ag_gemm_ex(p, TileShape(p.rows_per_rank(), p.local_cols()), [(a_shard, weight, out, pre)],
                    opts=N.default_opts(activation_grad=activation, b_layout=N.B_KN if b_kn else N.B_NK),
                    streams=_stream())
    return out


@ag_gemm_dact.register_fake
def _(a_shard, weight, pre, comm_id, activation, b_kn=False):
    n_local = weight.shape[1] if b_kn else weight.shape[0]
    width = n_local * (2 if activation == N.ACT_SWIGLU else 1)
    return a_shard.new_empty(a_shard.shape[0] * _REGISTRY[comm_id].tp, width)


def gathered_input(comm_id: int, a_shard: torch.Tensor, n_local: int) -> torch.Tensor:
    """Copy of this rank's gathered A of the last AG-GEMM (the symmetric a_agg)."""
    comm = _REGISTRY[comm_id]
    return comm.tensor(comm.rank, N.BUF_A_AGG, _ag_problem(comm, a_shard, n_local)).clone()


class _TPMlpFunction(torch.autograd.Function):
    """out = ReduceScatter(act(AllGather(x) W_up^T) W_down^T) with the fused
    operators; backward: dx = ReduceScatter((AllGather(dout) W_down) *
    act'(pre) W_up) (the AG <-> RS interchange), weight gradients as local
    GEMMs on the gathered operands read back from the symmetric heap."""

    @staticmethod
    def forward(ctx, x, w_up, w_down, comm_id, activation):
        z, pre = torch.ops.flux_b200.ag_gemm_act(x, w_up, comm_id, activation)
        x_g = gathered_input(comm_id, x, w_up.shape[0]) if w_up.requires_grad else None
        out = torch.ops.flux_b200.gemm_rs(z, w_down, comm_id)
        ctx.save_for_backward(w_up, w_down, z, pre, x_g)
        ctx.comm_id, ctx.activation = comm_id, activation
        return out

    @staticmethod
    def backward(ctx, dout):
        w_up, w_down, z, pre, x_g = ctx.saved_tensors
        dout = dout.contiguous().to(torch.bfloat16)
        # The backward GEMMs read the forward weights as [k, n] (MN-major B
        # operand): no transposed copies.
        dy = torch.ops.flux_b200.ag_gemm_dact(dout, w_down, pre, ctx.comm_id, ctx.activation, True)
        dout_g = gathered_input(ctx.comm_id, dout, w_down.shape[1]) if w_down.requires_grad else None
        dx = torch.ops.flux_b200.gemm_rs(dy, w_up, ctx.comm_id, True)
        d_w_up = (dy.t().float() @ x_g.float()).to(w_up.dtype) if x_g is not None else None
        d_w_down = (dout_g.t().float() @ z.float()).to(w_down.dtype) if dout_g is not None else None
        return dx, d_w_up, d_w_down, None, None


class TPMlp(torch.nn.Module):
    """Sequence-parallel tensor-parallel MLP block on the fused operators:
    x [m/tp, hidden] -> [m/tp, hidden]; w_up [ffn/tp (x2 SWIGLU), hidden],
    w_down [hidden, ffn/tp] (this rank's shards, nn.Linear layout)."""

    def __init__(self, hidden: int, ffn: int, comm_id: int, activation: int = N.ACT_GELU, device=None):
        super().__init__()
        tp = _REGISTRY[comm_id].tp
        rows = ffn // tp * (2 if activation == N.ACT_SWIGLU else 1)
        self.w_up = torch.nn.Parameter(torch.empty(rows, hidden, dtype=torch.bfloat16, device=device))
        self.w_down = torch.nn.Parameter(torch.empty(hidden, ffn // tp, dtype=torch.bfloat16, device=device))
        torch.nn.init.normal_(self.w_up, std=hidden ** -0.5)
        torch.nn.init.normal_(self.w_down, std=ffn ** -0.5)
        self.comm_id, self.activation = comm_id, activation

    def forward(self, x):
        return _TPMlpFunction.apply(x, self.w_up, self.w_down, self.comm_id, self.activation)
