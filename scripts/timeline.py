"""Device-trace timeline of one fused operator (profiling aid): events per
time bucket across all emulated ranks, from the kernel's %globaltimer trace.

    python scripts/timeline.py --workload llama70b-down-rs [--bucket-us 25]
"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N
from paper_2406_06858_b200.comm import read_trace
from bench import WORKLOADS

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="llama70b-down-rs")
ap.add_argument("--bucket-us", type=float, default=25.0)
ap.add_argument("--ag-engine", type=int, default=0)
ap.add_argument("--local", action="store_true", help="trace the plain local GEMM instead of the fused op")
ap.add_argument("--cta-ends", action="store_true", help="print the earliest / latest CTA end times with their ids")
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
for trace in (0, 0, 1):
    opts = fx.default_opts(trace=trace, ag_engine=args.ag_engine)
    comm.set_timing(True)
    if args.local:
        comm.local_gemm(prob, opts, streams=s)
    elif pattern == 0:
        comm.ag_gemm(prob, tile, prob.rows_per_rank(), fx.PULL, True, opts, streams=s)
    else:
        comm.gemm_rs(prob, tile, fx.WRITE_ALLTOALL, True, opts, streams=s)
    comm.sync()
    print(f"trace={trace} kernel {comm.last_kernel_ms():.4f} ms")
ev = []
for r in range(tp):
    ev += read_trace(comm, r, prob)
t0 = min(e["ts"] for e in ev)
b = args.bucket_us * 1000
hist = collections.defaultdict(collections.Counter)
for e in ev:
    hist[int((e["ts"] - t0) // b)][e["event"]] += 1
kinds = sorted({e["event"] for e in ev})
print("t_us      " + " ".join(f"{x:>14s}" for x in kinds))
for i in sorted(hist):
    print(f"{i * args.bucket_us:8.1f}  " + " ".join(f"{hist[i][x]:14d}" for x in kinds))
print(f"span {(max(e['ts'] for e in ev) - t0) / 1000:.1f} us, {len(ev)} events")
starts = [e["ts"] for e in ev if e["event"] == "launch" and e["tile_col"] == 0]
ends = [e["ts"] for e in ev if e["event"] == "launch" and e["tile_col"] == 1]
if starts and ends:
    print(f"CTAs: first start -> last start {(max(starts) - min(starts)) / 1e3:.1f} us, first start -> last end "
          f"{(max(ends) - min(starts)) / 1e3:.1f} us (kernel event time above includes launch + teardown)")
    ends_us = sorted((e - min(starts)) / 1e3 for e in ends)
    q = [ends_us[int(f * (len(ends_us) - 1))] for f in (0.0, 0.1, 0.5, 0.9, 1.0)]
    print("CTA end times (us) min/p10/p50/p90/max: " + " / ".join(f"{v:.1f}" for v in q))
    if args.cta_ends:
        t00 = min(starts)
        by = sorted(((e["ts"] - t00) / 1e3, e["tile_row"]) for e in ev if e["event"] == "launch" and e["tile_col"] == 1)
        print("earliest CTA ends (us, blockIdx):", [(round(t), b) for t, b in by[:16]])
        print("latest CTA ends (us, blockIdx):", [(round(t), b) for t, b in by[-16:]])
