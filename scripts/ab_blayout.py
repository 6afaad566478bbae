"""A/B of the B operand layout on one workload: caller B as [n, k] (K-major)
vs [k, n] row-major (opts.b_layout = KN, MN-major tcgen05 operand), round-robin
medians (profiling aid)."""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N
from bench import WORKLOADS

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="llama70b-up-ag")
ap.add_argument("--rounds", type=int, default=12)
args = ap.parse_args()
pattern, m, n, k, tp, _ = WORKLOADS[args.workload]
p = fx.ProblemSpec(m, n, k, tp, pattern)
cs = torch.cuda.Stream()
torch.cuda.set_stream(cs)
comm = fx.Communicator(tp, [0] * tp, heap_bytes=fx.required_heap_bytes(p) + (64 << 20))
for r in range(tp):
    for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
        t = comm.tensor(r, kind, p)
        t.copy_(torch.rand(t.shape, device="cuda").mul_(2).sub_(1))
b_nk = [comm.tensor(r, N.BUF_B_SHARD, p).clone() for r in range(tp)]
b_kn = [t.t().contiguous() for t in b_nk]
st = [cs.cuda_stream] * tp
tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def run(bs, layout):
    o = fx.default_opts(b_layout=layout)
    ops = [(None, bs[r], None) for r in range(tp)]
    if pattern == fx.ALLGATHER_GEMM:
        comm.ag_gemm_ex(p, tile, ops, opts=o, streams=st)
    else:
        comm.gemm_rs_ex(p, tile, ops, opts=o, streams=st)


cfgs = {"B [n, k] (K-major)": (b_nk, fx.B_NK), "B [k, n] (MN-major)": (b_kn, fx.B_KN)}
for bs, lay in cfgs.values():
    run(bs, lay)
torch.cuda.synchronize()
times = {name: [] for name in cfgs}
for _ in range(args.rounds):
    for name, (bs, lay) in cfgs.items():
        flush.zero_()
        e0.record(cs)
        run(bs, lay)
        e1.record(cs)
        e1.synchronize()
        times[name].append(e0.elapsed_time(e1))
for name, ts in times.items():
    print(f"{args.workload} {name:24s} median {statistics.median(ts) * 1e3:8.1f} us  min {min(ts) * 1e3:8.1f}")
