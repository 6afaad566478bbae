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
    p = ProblemSpec(a_shard.shape[0] * tp, weight.shape[0] * tp, k, tp, N.ALLGATHER_GEMM)
    out = torch.empty(p.m, weight.shape[0], dtype=torch.bfloat16, device=a_shard.device)
    comm.ag_gemm_ex(p, TileShape(p.rows_per_rank(), p.local_cols()), [(a_shard, weight, out)], streams=_stream())
    return out


@ag_gemm.register_fake
def _(a_shard, weight, comm_id):
    return a_shard.new_empty(a_shard.shape[0] * _REGISTRY[comm_id].tp, weight.shape[0])


@torch.library.custom_op("flux_b200::gemm_rs", mutates_args=())
def gemm_rs(a: torch.Tensor, weight: torch.Tensor, comm_id: int) -> torch.Tensor:
    """ReduceScatter(a @ weight^T) over rows. a [m, k/tp] bf16, weight [n, k/tp]
    bf16; returns this rank's [m/tp, n] bf16 rows (source-ordered fp32 sum)."""
    comm = _REGISTRY[comm_id]
    tp = comm.tp
    p = ProblemSpec(a.shape[0], weight.shape[0], a.shape[1] * tp, tp, N.GEMM_REDUCESCATTER)
    aligned = p.rows_per_rank() % 128 == 0
    out = torch.empty(p.rows_per_rank(), p.n, dtype=torch.bfloat16, device=a.device) if aligned else None
    comm.gemm_rs_ex(p, TileShape(p.rows_per_rank(), p.local_cols()), [(a, weight, out)], streams=_stream())
    if out is None:  # decode-sized blocks: the result lives in the symmetric heap
        out = comm.tensor(comm.rank, N.BUF_C_OUT, p).clone()
    return out


@gemm_rs.register_fake
def _(a, weight, comm_id):
    return a.new_empty(a.shape[0] // _REGISTRY[comm_id].tp, weight.shape[0])
