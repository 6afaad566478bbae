"""A/B of the AllGather transfer engines (copy engines vs in-kernel TMA bulk
copies) on one workload, alternating one step of each per round (medians),
so clock/power drift biases neither (profiling aid)."""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N
from paper_2406_06858_b200 import tune as T
from bench import WORKLOADS

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="llama70b-up-ag")
ap.add_argument("--rounds", type=int, default=12)
args = ap.parse_args()
pattern, m, n, k, tp, _ = WORKLOADS[args.workload]
p = fx.ProblemSpec(m, n, k, tp, pattern)
torch.cuda.set_stream(torch.cuda.Stream())
comm = fx.Communicator(tp, [0] * tp, heap_bytes=fx.required_heap_bytes(p) + (64 << 20))
for r in range(tp):
    for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
        t = comm.tensor(r, kind, p)
        t.copy_(torch.rand(t.shape, device="cuda").mul_(2).sub_(1))
torch.cuda.synchronize()
meas = T.gpu_measure(comm, p, 1)
tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
cfgs = {"copy": T.TuneConfig(tile, fx.SWIZZLE_ARRIVAL_ALIGNED, p.rows_per_rank(), fx.PULL, ag_engine=1),
        "sm": T.TuneConfig(tile, fx.SWIZZLE_ARRIVAL_ALIGNED, p.rows_per_rank(), fx.PULL, ag_engine=2),
        "auto": T.TuneConfig(tile, fx.SWIZZLE_ARRIVAL_ALIGNED, p.rows_per_rank(), fx.PULL, ag_engine=0)}
times = {k: [] for k in cfgs}
for _ in range(args.rounds):
    for name, c in cfgs.items():
        times[name] += meas(c)
for name, ts in times.items():
    print(f"{args.workload} engine={name}: median {statistics.median(ts):.1f} us  min {min(ts):.1f}")
