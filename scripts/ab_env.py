"""Round-robin A/B of library settings read from the environment at each call
(FLUX_GROUP_BLOCKS, FLUX_RS_CHAIN, ...) or of opts fields, one step of each
configuration per round, L2 flushed before each, medians over the rounds — so
clock / power drift biases no configuration (profiling aid).

    python scripts/ab_env.py --workload llama70b-up-ag --cfg "" --cfg FLUX_GROUP_BLOCKS=2 --cfg opt:ag_engine=2,push=1
"""
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
ap.add_argument("--rounds", type=int, default=20)
ap.add_argument("--cfg", action="append", default=[])
ap.add_argument("--local", action="store_true", help="also time the plain local GEMM each round")
ap.add_argument("--op", default="fused", choices=["fused", "local"], help="what each --cfg runs")
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
st = [torch.cuda.current_stream().cuda_stream] * tp
tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def make(cfg):
    env, opt = {}, {}
    push = False
    for kv in filter(None, cfg.split(",")):
        key, val = kv.split("=", 1)
        if key == "push":  # AllGather transfer mode
            push = val == "1"
        elif key.startswith("opt:"):
            opt[key[4:]] = int(val)
        else:
            env[key] = val

    def run():
        saved = {key: os.environ.get(key) for key in env}
        os.environ.update(env)
        o = fx.default_opts(**opt)
        if args.op == "local":
            comm.local_gemm(p, o, st)
        elif pattern == fx.ALLGATHER_GEMM:
            comm.ag_gemm(p, tile, p.rows_per_rank(), fx.PUSH if push else fx.PULL, True, o, st)
        else:
            comm.gemm_rs(p, tile, fx.WRITE_ALLTOALL, True, o, st)
        for key, old in saved.items():
            if old is None:
                os.environ.pop(key, None)
            else:
                os.environ[key] = old
    return run


fns = {cfg or "default": make(cfg) for cfg in (args.cfg or [""])}
if args.local:
    fns["local GEMM"] = lambda: comm.local_gemm(p, None, st)
for fn in fns.values():
    fn()
    fn()
torch.cuda.synchronize()
times = {name: [] for name in fns}
for _ in range(args.rounds):
    for name, fn in fns.items():
        flush.zero_()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        times[name].append(e0.elapsed_time(e1))
comm.sync()
base = statistics.median(next(iter(times.values())))
for name, ts in times.items():
    med = statistics.median(ts)
    print(f"{args.workload} {name:40s} median {med * 1e3:8.1f} us  min {min(ts) * 1e3:8.1f}  vs first {med / base:.3f}")
