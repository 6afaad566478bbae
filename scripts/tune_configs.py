"""Runs the GPU-calibrated autotuner (paper_2406_06858_b200/tune.py) on the
BASELINE.json workloads (ranks emulated on one GPU) and writes the reference
tuner's reports: <out>/<workload>.csv / .json and the cache file.

    python scripts/tune_configs.py [--out profiles/round1/tune] [--reps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N
from paper_2406_06858_b200 import tune as T
from bench import WORKLOADS

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="profiles/round1/tune")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--workloads", default="llama70b-up-ag,llama70b-down-rs,decode-ag-m64,decode-rs-m64")
args = ap.parse_args()
os.makedirs(args.out, exist_ok=True)
extra = {"decode-ag-m64": (0, 64, 28672, 8192, 8, ""), "decode-rs-m64": (1, 64, 8192, 28672, 8, "")}
torch.cuda.set_stream(torch.cuda.Stream())
summary = {}
for wl in args.workloads.split(","):
    pattern, m, n, k, tp, _ = {**WORKLOADS, **extra}[wl]
    p = fx.ProblemSpec(m, n, k, tp, pattern)
    comm = fx.Communicator(tp, [0] * tp, heap_bytes=fx.required_heap_bytes(p) + (64 << 20))
    for r in range(tp):
        for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
            t = comm.tensor(r, kind, p)
            t.copy_(torch.rand(t.shape, device="cuda").mul_(2).sub_(1))
    torch.cuda.synchronize()
    ks = T.default_knob_space(p)
    # The device tile is fixed (128x256 / 256x256); (tm, tn) only sets the
    # ownership and comm granularity, so one tile shape spans the comm sizes.
    ks.gemm_tile_shapes = [fx.TileShape(min(64, p.rows_per_rank()), min(128, p.local_cols()))]
    res = T.tune(p, ks, T.gpu_measure(comm, p, args.reps), T.gpu_verify(comm, p), repetitions=args.reps,
                 cache_path=os.path.join(args.out, f"{wl}.cache.json"), machine=T.machine_id())
    T.write_tune_csv(os.path.join(args.out, f"{wl}.csv"), res)
    T.write_tune_json(os.path.join(args.out, f"{wl}.json"), res)
    # The library's automatic choice (what bench.py runs) for comparison.
    default = T.TuneConfig(fx.TileShape(p.rows_per_rank(), p.local_cols()),
                           fx.SWIZZLE_RANK_SHIFTED if pattern else fx.SWIZZLE_ARRIVAL_ALIGNED,
                           p.rows_per_rank(), fx.PULL, fx.WRITE_ALLTOALL if pattern else fx.FUSED_REDUCE)
    d = sorted(T.gpu_measure(comm, p, max(5, args.reps))(default))
    summary[wl] = {"configs": len(res.table), "best": res.best_config.encode(), "best_us": res.objective_us,
                   "default_us": d[len(d) // 2], "default_vs_best": d[len(d) // 2] / res.objective_us}
    print(wl, json.dumps(summary[wl]), flush=True)
    comm.close()
    torch.cuda.empty_cache()
json.dump(summary, open(os.path.join(args.out, "summary.json"), "w"), indent=1)
