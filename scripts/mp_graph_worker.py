"""One rank of a two-process CUDA-graph run (launched by
tests/test_multiprocess_gpu.py with torchrun, gloo for the host exchanges):
graph-safe fused operators on the one-process-per-GPU (IPC) communicator are
captured once and replayed on new inputs, with eager operators in between; the
device-side rank barriers that bracket a graph-safe operator replace the eager
operators' host stream memops. Every replay and every eager operator is checked
against the oracle. The first operator on each communicator is graph-safe (no
eager epoch stamps exist yet)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N
from oracle import oracle as O

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = rank % torch.cuda.device_count()
torch.cuda.set_device(dev)
dist.init_process_group("gloo")


def gather(blob):
    out = [None] * world
    dist.all_gather_object(out, blob)
    return out


def upload(comm, p, seed):
    a_bits, bt_bits = O.rank_inputs_bits(p.pattern, p.m, p.n, p.k, world, seed, rank)
    comm.tensor(rank, N.BUF_A_SHARD, p).copy_(torch.from_numpy(a_bits.view(np.int16)).cuda().view(torch.bfloat16))
    comm.tensor(rank, N.BUF_B_SHARD, p).copy_(torch.from_numpy(bt_bits.view(np.int16)).cuda().view(torch.bfloat16))
    torch.cuda.synchronize()


def check(comm, p, seed):
    got = comm.tensor(rank, N.BUF_C_OUT_F32, p).double().cpu().numpy()
    ins = [O.rank_inputs(p.pattern, p.m, p.n, p.k, world, seed, r) for r in range(world)]
    want = O.dense_oracle(p.pattern, p.m, p.n, p.k, world, [x[0] for x in ins], [x[1] for x in ins])[rank]
    return O.max_rel_error(got, want)


def op(comm, p, opts, streams=None):
    tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
    if p.pattern == fx.ALLGATHER_GEMM:
        comm.ag_gemm(p, tile, p.rows_per_rank(), fx.PULL, True, opts, streams)
    else:
        comm.gemm_rs(p, tile, fx.WRITE_ALLTOALL, True, opts, streams)


cases = [(fx.ALLGATHER_GEMM, 256 * world, 512 * world, 512), (fx.GEMM_REDUCESCATTER, 256 * world, 512, 256 * world),
         (fx.GEMM_REDUCESCATTER, 16 * world, 1024, 512 * world), (fx.ALLGATHER_GEMM, 16 * world, 1024 * world, 512)]
results = {}
side = torch.cuda.Stream()
streams = [side.cuda_stream]
gopts = fx.default_opts(out_dtype=fx.F32, graph_safe=1, wall_budget_s=20.0)
eopts = fx.default_opts(out_dtype=fx.F32, wall_budget_s=20.0)
for pat, m, n, k in cases:
    p = fx.ProblemSpec(m, n, k, world, pat)
    comm = fx.Communicator.ipc(rank, world, dev, fx.required_heap_bytes(p) + (8 << 20), gather)
    tol = 1e-4 * max(1.0, k / 1024.0)
    errs = []
    upload(comm, p, 11)
    dist.barrier()
    with torch.cuda.stream(side):
        op(comm, p, gopts, streams)  # first operator of the communicator: graph-safe, eager launch
    comm.sync()
    errs.append(check(comm, p, 11))
    dist.barrier()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        op(comm, p, gopts, streams)
    dist.barrier()
    for it in range(5):
        seed = 100 + it
        upload(comm, p, seed)
        if it in (2, 3):  # eager operators between replays (epoch-stamped flags, host memops)
            dist.barrier()
            op(comm, p, eopts)
            comm.sync()
            errs.append(check(comm, p, seed))
            dist.barrier()
        graph.replay()  # no host barrier: the replay's device barriers order it against the peer
        torch.cuda.synchronize()
        errs.append(check(comm, p, seed))
        dist.barrier()  # the peer may still read this rank's inputs
    upload(comm, p, 7)
    dist.barrier()
    op(comm, p, eopts)
    comm.sync()
    errs.append(check(comm, p, 7))
    del graph
    comm.close()
    results[f"{pat} {m}x{n}x{k}"] = (max(errs), tol, len(errs))
    dist.barrier()
for r in range(world):
    if r == rank:
        print(f"RESULT {rank} {json.dumps(results)}", flush=True)
    dist.barrier()
dist.destroy_process_group()
