"""Eager vs CUDA-graph replay of back-to-back fused operators (decode shapes,
ranks emulated on one GPU): per-operator device time of a burst of `--ops`
operators issued eagerly (default opts, and graph_safe) and replayed from one
captured graph. Prints one JSON line per workload.

    python scripts/graph_bench.py --workloads decode-ag-up-m16,decode-rs-down-m16
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N
from bench import WORKLOADS

ap = argparse.ArgumentParser()
ap.add_argument("--workloads", default="decode-ag-up-m16,decode-rs-down-m16,decode-rs-attn-m16")
ap.add_argument("--ops", type=int, default=20)
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()
side = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

for name in args.workloads.split(","):
    pattern, m, n, k, tp, _ = WORKLOADS[name]
    p = fx.ProblemSpec(m, n, k, tp, pattern)
    tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
    st = [side.cuda_stream] * tp
    with fx.Communicator(tp, [0] * tp, heap_bytes=fx.required_heap_bytes(p) + (64 << 20)) as comm:
        for r in range(tp):
            for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
                t = comm.tensor(r, kind, p)
                t.copy_(torch.rand(t.shape, device="cuda").mul_(2).sub_(1))
        torch.cuda.synchronize()

        def op(opts):
            if pattern == fx.ALLGATHER_GEMM:
                comm.ag_gemm(p, tile, p.rows_per_rank(), fx.PULL, True, opts, st)
            else:
                comm.gemm_rs(p, tile, fx.WRITE_ALLTOALL, True, opts, st)

        def burst(opts):
            for _ in range(args.ops):
                op(opts)

        res = {"workload": name, "ops_per_burst": args.ops}
        eager, gsafe = fx.default_opts(), fx.default_opts(graph_safe=1)
        with torch.cuda.stream(side):
            for label, o in (("eager", eager), ("eager_graph_safe", gsafe)):
                burst(o)
                side.synchronize()
                dev, host = [], []
                for _ in range(args.reps):
                    e0.record(side)
                    t0 = time.perf_counter()
                    burst(o)
                    host.append((time.perf_counter() - t0) / args.ops * 1e6)
                    e1.record(side)
                    e1.synchronize()
                    dev.append(e0.elapsed_time(e1) / args.ops * 1e3)
                res[label + "_us_per_op"] = sorted(dev)[len(dev) // 2]
                res[label + "_host_us_per_op"] = sorted(host)[len(host) // 2]
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            burst(gsafe)
        graph.replay()
        torch.cuda.synchronize()
        dev = []
        for _ in range(args.reps):
            e0.record(side)
            with torch.cuda.stream(side):
                graph.replay()
            e1.record(side)
            e1.synchronize()
            dev.append(e0.elapsed_time(e1) / args.ops * 1e3)
        res["graph_replay_us_per_op"] = sorted(dev)[len(dev) // 2]
        comm.sync()
        print(json.dumps(res), flush=True)
