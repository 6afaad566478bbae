"""Kernel-time ablations of one workload's fused operator (profiling aid).

    python scripts/ablate.py --workload llama70b-down-rs --env FLUX_DEBUG=1 --env FLUX_DEBUG=2 ...

Each `--env` entry (comma-separated KEY=VAL pairs) is one configuration; the
baseline (no overrides) always runs first. Prints mean kernel ms per config.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N
from bench import WORKLOADS

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="llama70b-down-rs")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--env", action="append", default=[])
ap.add_argument("--op", default="fused", choices=["fused", "local"])
ap.add_argument("--ag-engine", type=int, default=0)
ap.add_argument("--cta-group", type=int, default=0)
ap.add_argument("--write-mode", type=int, default=0)
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
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
opts = fx.default_opts(ag_engine=args.ag_engine, cta_group=args.cta_group,
                       deterministic_reduce=0 if args.write_mode == 1 else 1)


def run(op=None):
    if (op or args.op) == "local":
        comm.local_gemm(prob, opts, streams=s)
    elif pattern == 0:
        comm.ag_gemm(prob, tile, prob.rows_per_rank(), fx.PULL, True, opts, streams=s)
    else:
        comm.gemm_rs(prob, tile, args.write_mode, True, opts, streams=s)


def local_ms():
    comm.set_timing(True)
    ms = []
    for i in range(args.iters + 3):
        flush.fill_(i & 0xFF)
        run("local")
        comm.sync()
        if i >= 3:
            ms.append(comm.last_kernel_ms())
    comm.set_timing(False)
    return statistics.mean(ms)


ref = local_ms()
print(f"{args.workload} local GEMM (plain kernel, reference) {ref:.4f} ms", flush=True)
results = {}
for cfg in [""] + args.env:
    saved = {}
    for kv in filter(None, cfg.split(",")):
        key, val = kv.split("=", 1)
        saved[key] = os.environ.get(key)
        os.environ[key] = val
    comm.set_timing(True)
    ms = []
    for i in range(args.iters + 3):
        flush.fill_(i & 0xFF)
        run()
        comm.sync()
        if i >= 3:
            ms.append(comm.last_kernel_ms())
    comm.set_timing(False)
    for key, old in saved.items():
        if old is None:
            os.environ.pop(key, None)
        else:
            os.environ[key] = old
    results[cfg or "baseline"] = (statistics.mean(ms), min(ms))
    print(f"{args.workload} {cfg or 'baseline':40s} kernel mean {statistics.mean(ms):.4f} ms  min {min(ms):.4f} ms"
          f"  ratio to local {statistics.mean(ms) / ref:.3f}", flush=True)
ref2 = local_ms()
print(f"{args.workload} local GEMM again {ref2:.4f} ms (drift {ref2 / ref - 1:+.1%})", flush=True)
print(json.dumps({k: v[0] for k, v in results.items()}))
