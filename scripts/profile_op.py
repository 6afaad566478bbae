"""Runs one workload's fused operator a few times (for ncu captures)."""
import argparse
import sys

sys.path.insert(0, ".")
import torch

import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N
from bench import WORKLOADS

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="llama70b-up-ag")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--op", default="fused", choices=["fused", "local", "nonoverlap"])
args = ap.parse_args()
pattern, m, n, k, tp, _ = WORKLOADS[args.workload]
prob = fx.ProblemSpec(m, n, k, tp, pattern)
torch.cuda.set_stream(torch.cuda.Stream())
comm = fx.Communicator(tp, [0] * tp, heap_bytes=fx.required_heap_bytes(prob) + (64 << 20))
for r in range(tp):
    for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
        t = comm.tensor(r, kind, prob)
        t.copy_(torch.rand(t.shape, device="cuda").mul_(2).sub_(1))
torch.cuda.synchronize()
s = [torch.cuda.current_stream().cuda_stream] * tp
tile = fx.TileShape(prob.rows_per_rank(), prob.local_cols())
for _ in range(args.iters):
    if args.op == "local":
        comm.local_gemm(prob, streams=s)
    elif args.op == "nonoverlap":
        comm.nonoverlap(prob, streams=s)
    elif pattern == 0:
        comm.ag_gemm(prob, tile, prob.rows_per_rank(), fx.PULL, True, streams=s)
    else:
        comm.gemm_rs(prob, tile, fx.WRITE_ALLTOALL, True, streams=s)
comm.sync()
print("done")
