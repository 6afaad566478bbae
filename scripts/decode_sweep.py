"""Decode-regime sweep (BASELINE.json configs[4]): M = 16..512 tokens at TP=8
(emulated on one GPU) for Llama-2-70B AG up-proj (K=8192, N=28672), RS
down-proj (K=28672, N=8192) and RS attention-out (K=8192, N=8192). Reports the
fused operator latency, the unfused baseline (copies + cuBLAS) and the HBM
roofline (the weights must be streamed once)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N
from paper_2406_06858_b200 import baselines as BL

ap = argparse.ArgumentParser()
ap.add_argument("--ms", default="16,32,64,128,256,512")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--out", default="")
args = ap.parse_args()
torch.cuda.set_stream(torch.cuda.Stream())
st = torch.cuda.current_stream().cuda_stream
HBM = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
# TP=8 emulated on one GPU (every rank's work in one launch), and one GPU's
# share at TP=8 (tp=1 problems with the per-rank shapes: what one GPU streams).
shapes = {"ag-up": (0, 28672, 8192, 8), "rs-down": (1, 8192, 28672, 8), "rs-attn-out": (1, 8192, 8192, 8),
          "rank-ag-up": (0, 3584, 8192, 1), "rank-rs-down": (1, 8192, 3584, 1), "rank-rs-attn-out": (1, 8192, 1024, 1)}
ap2 = [x for x in os.environ.get("SWEEP_SHAPES", "").split(",") if x]
if ap2:
    shapes = {k: v for k, v in shapes.items() if k in ap2}
rows = []
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(64 << 20, dtype=torch.int32, device="cuda")  # read sweep: no dirty lines left in L2


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(args.iters):
        flush.zero_()
        flush_rd.max()
        e0.record(); fn(); e1.record(); e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / args.iters


for name, (pat, n, k, tp) in shapes.items():
    for m in [int(x) for x in args.ms.split(",")]:
        p = fx.ProblemSpec(m, n, k, tp, pat)
        comm = fx.Communicator(tp, [0] * tp, heap_bytes=fx.required_heap_bytes(p) + (16 << 20))
        for r in range(tp):
            for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
                t = comm.tensor(r, kind, p)
                t.copy_(torch.rand(t.shape, device="cuda").mul_(2).sub_(1))
        tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
        streams = [st] * tp
        if pat == 0:
            fused = lambda: comm.ag_gemm(p, tile, p.rows_per_rank(), fx.PULL, True, None, streams)
            b = BL.EmulatedAG([comm.tensor(r, N.BUF_A_SHARD, p).contiguous() for r in range(tp)],
                              [comm.tensor(r, N.BUF_B_SHARD, p).contiguous() for r in range(tp)])
        else:
            fused = lambda: comm.gemm_rs(p, tile, fx.WRITE_ALLTOALL, True, None, streams)
            b = BL.EmulatedRS([comm.tensor(r, N.BUF_A_SHARD, p).contiguous() for r in range(tp)],
                              [comm.tensor(r, N.BUF_B_SHARD, p).contiguous() for r in range(tp)])
        t_fused = timed(fused)
        comm.sync()
        comm.set_timing(True)
        kms = []
        for _ in range(5):
            fused()
            kms.append(comm.last_kernel_ms())
        comm.set_timing(False)
        comm.sync()
        t_b1 = timed(b.unfused)
        t_local = timed(lambda: comm.local_gemm(p, None, streams))  # the same GEMMs, no communication
        wbytes = 2.0 * n * k  # all ranks' weight shards, streamed once
        row = {"shape": name, "m": m, "tp": tp, "fused_ms": t_fused, "kernel_ms": sorted(kms)[len(kms) // 2],
               "unfused_ms": t_b1, "local_gemm_ms": t_local, "overhead_vs_local": t_fused / t_local - 1.0,
               "speedup": t_b1 / t_fused, "hbm_roofline_ms": wbytes / (HBM * 1e9) * 1e3,
               "roofline_frac": (wbytes / (HBM * 1e9) * 1e3) / t_fused}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del b
        comm.close()
        torch.cuda.empty_cache()
if args.out:
    json.dump(rows, open(args.out, "w"), indent=1)
