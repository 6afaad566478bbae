"""Chained tensor-parallel MLP forward on the BASELINE
shapes, ranks emulated on one GPU: flux_mlp_forward (AG-GEMM with the
activation in its epilogue -> GEMM-RS on the intermediate) against the
unfused chain (device copies for the all-gather, cuBLAS GEMMs, the activation
as separate torch kernels, device adds for the reduce-scatter). Round-robin
medians, L2 flushed before each step.

    python scripts/mlp_bench.py [--model llama70b|gpt3] [--m 4096] [--tp 8]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2406_06858_b200 as fx

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama70b", choices=["llama70b", "gpt3"])
ap.add_argument("--m", type=int, default=4096)
ap.add_argument("--tp", type=int, default=8)
ap.add_argument("--rounds", type=int, default=10)
args = ap.parse_args()
hidden, ffn, act = (8192, 28672, fx.ACT_SWIGLU) if args.model == "llama70b" else (12288, 49152, fx.ACT_GELU)
tp, m = args.tp, args.m
f, rpr = ffn // tp, m // tp
glu = act == fx.ACT_SWIGLU
spec = fx.MlpSpec(m, hidden, ffn, tp, act)
torch.cuda.set_stream(torch.cuda.Stream())
dev = "cuda"
g = torch.Generator(device=dev)
g.manual_seed(0)


def rnd(*shape, scale=1.0):
    return ((torch.rand(*shape, generator=g, device=dev) * 2 - 1) * scale).to(torch.bfloat16)


x = [rnd(rpr, hidden) for _ in range(tp)]
w_up = [rnd(2 * f if glu else f, hidden, scale=0.02) for _ in range(tp)]
w_down = [rnd(hidden, f, scale=0.02) for _ in range(tp)]
inter = [torch.empty(m, f, dtype=torch.bfloat16, device=dev) for _ in range(tp)]
out = [torch.empty(rpr, hidden, dtype=torch.bfloat16, device=dev) for _ in range(tp)]
comm = fx.Communicator(tp, [0] * tp, heap_bytes=spec.required_heap_bytes())
st = [torch.cuda.current_stream().cuda_stream] * tp
ops = [dict(x=x[r], w_up=w_up[r], w_down=w_down[r], act=inter[r], out=out[r]) for r in range(tp)]

# unfused chain buffers
gathered = torch.empty(m, hidden, dtype=torch.bfloat16, device=dev)
y_full = torch.empty(m, w_up[0].shape[0], dtype=torch.bfloat16, device=dev)
partials = [torch.empty(m, hidden, dtype=torch.bfloat16, device=dev) for _ in range(tp)]
out_ref = [torch.empty(rpr, hidden, dtype=torch.bfloat16, device=dev) for _ in range(tp)]


def fused():
    comm.mlp_forward(spec, ops, streams=st)


def unfused():
    for r in range(tp):
        for q in range(tp):  # all-gather: tp device copies into this rank's buffer
            gathered[q * rpr:(q + 1) * rpr].copy_(x[q])
        torch.matmul(gathered, w_up[r].t(), out=y_full)
        if glu:
            y4 = y_full.view(m, -1, 2, 128)
            z = torch.nn.functional.silu(y4[:, :, 0]) * y4[:, :, 1]
            z = z.reshape(m, -1)
        else:
            z = torch.nn.functional.gelu(y_full)
        torch.matmul(z, w_down[r].t(), out=partials[r])
    for r in range(tp):  # reduce-scatter: sum the partials' row blocks in rank order
        acc = partials[0][r * rpr:(r + 1) * rpr].float()
        for s in range(1, tp):
            acc += partials[s][r * rpr:(r + 1) * rpr]
        out_ref[r].copy_(acc)


flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
fns = {"fused": fused, "unfused": unfused}
for fn in fns.values():
    fn()
torch.cuda.synchronize()
times = {k: [] for k in fns}
for _ in range(args.rounds):
    for name, fn in fns.items():
        flush.zero_()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        times[name].append(e0.elapsed_time(e1))
comm.sync()
err = max(((out[r].float() - out_ref[r].float()).abs().max() / out_ref[r].float().abs().max()).item() for r in range(tp))
flops = 2.0 * m * hidden * (2 * ffn if glu else ffn) + 2.0 * m * ffn * hidden
res = {"model": args.model, "m": m, "tp": tp, "activation": "swiglu" if glu else "gelu",
       "fused_ms": statistics.median(times["fused"]), "unfused_ms": statistics.median(times["unfused"]),
       "max_rel_diff_vs_unfused": err}
res["fused_tflops"] = flops / (res["fused_ms"] * 1e-3) / 1e12
res["unfused_tflops"] = flops / (res["unfused_ms"] * 1e-3) / 1e12
res["speedup"] = res["unfused_ms"] / res["fused_ms"]
print(json.dumps(res), flush=True)
comm.close()
