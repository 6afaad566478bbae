"""One rank of a two-process NVLS run (launched by tests/test_multiprocess_gpu.py
with torchrun, gloo for the exchanges): sets up the IPC communicator with an
NVLS region — rank 0's multicast handle reaches the peer as a file descriptor
over a Unix socket — and, where the host exposes multicast, checks the
multicast AllGather-GEMM / GEMM-RS against the oracle; otherwise every rank
must raise the same error. The emulated NVLS protocol (unicast loops over the
peers' IPC-mapped regions) is checked against the oracle either way."""
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


cases = [(fx.ALLGATHER_GEMM, 256 * world, 512 * world, 512), (fx.GEMM_REDUCESCATTER, 256 * world, 512, 256 * world),
         (fx.GEMM_REDUCESCATTER, 16 * world, 1024, 512 * world)]
probs = [fx.ProblemSpec(m, n, k, world, pat) for pat, m, n, k in cases]
heap = max(fx.required_heap_bytes(p) for p in probs) + (8 << 20)
nvls_bytes = max(fx.nvls_required_bytes(p) for p in probs)
results, mc = {}, "unavailable"
try:
    comm = fx.Communicator.ipc(rank, world, dev, heap, gather, nvls_bytes=nvls_bytes)
    mc = "ok"
except fx.FluxError as e:
    mc = "error: " + str(e)
    comm = fx.Communicator.ipc(rank, world, dev, heap, gather)


def run(p, nvls):
    a_bits, bt_bits = O.rank_inputs_bits(p.pattern, p.m, p.n, p.k, world, 3, rank)
    comm.tensor(rank, N.BUF_A_SHARD, p).copy_(torch.from_numpy(a_bits.view(np.int16)).cuda().view(torch.bfloat16))
    comm.tensor(rank, N.BUF_B_SHARD, p).copy_(torch.from_numpy(bt_bits.view(np.int16)).cuda().view(torch.bfloat16))
    torch.cuda.synchronize()
    dist.barrier()
    opts = fx.default_opts(out_dtype=fx.F32, wall_budget_s=20.0, nvls=nvls)
    tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
    for _ in range(2):
        if p.pattern == fx.ALLGATHER_GEMM:
            comm.ag_gemm(p, tile, p.rows_per_rank() // 2, fx.PULL, True, opts)
        else:
            comm.gemm_rs(p, tile, fx.WRITE_ALLTOALL, True, opts)
        comm.sync()
    got = comm.tensor(rank, N.BUF_C_OUT_F32, p).double().cpu().numpy()
    ins = [O.rank_inputs(p.pattern, p.m, p.n, p.k, world, 3, r) for r in range(world)]
    want = O.dense_oracle(p.pattern, p.m, p.n, p.k, world, [x[0] for x in ins], [x[1] for x in ins])[rank]
    dist.barrier()
    return O.max_rel_error(got, want), 1e-4 * max(1.0, p.k / 1024.0)


for p in probs:
    results[f"emulated {p.pattern} {p.m}x{p.n}x{p.k}"] = run(p, fx.NVLS_EMULATED)
    if mc == "ok":
        results[f"multicast {p.pattern} {p.m}x{p.n}x{p.k}"] = run(p, fx.NVLS_MULTICAST)
comm.close()
for r in range(world):
    if r == rank:
        print(f"RESULT {rank} {json.dumps({'multicast': mc, 'results': results})}", flush=True)
    dist.barrier()
dist.destroy_process_group()
