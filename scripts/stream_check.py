"""Profiling aid: the streaming decode kernel (flux_opts.decode_kernel) against
the tile kernel on decode shapes — outputs compared with each other and with a
torch fp32 product of the same bf16 operands, and per-op device time (L2
flushed between ops: 256 MiB write, then a 256 MiB read sweep).

    python scripts/stream_check.py [shape ...]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2406_06858_b200 as fx  # noqa: E402
from paper_2406_06858_b200 import _native as N  # noqa: E402

# name: (pattern, m, n, k, tp) — tp=1: one GPU's share of the TP=8 decode step
SHAPES = {
    "rank-ag-up-m16": (0, 16, 3584, 8192, 1), "rank-rs-down-m16": (1, 16, 8192, 3584, 1),
    "rank-rs-attn-m16": (1, 16, 8192, 1024, 1), "rank-ag-up-m128": (0, 128, 3584, 8192, 1),
    "rank-rs-down-m128": (1, 128, 8192, 3584, 1), "rank-ag-up-m64": (0, 64, 3584, 8192, 1),
    "ag-up-m16-tp8": (0, 16, 28672, 8192, 8), "rs-down-m16-tp8": (1, 16, 8192, 28672, 8),
    "rs-attn-m16-tp8": (1, 16, 8192, 8192, 8), "ag-up-m128-tp8": (0, 128, 28672, 8192, 8),
    "rs-down-m128-tp8": (1, 128, 8192, 28672, 8), "rs-attn-m128-tp8": (1, 128, 8192, 8192, 8),
}
dev = torch.device("cuda", 0)
torch.cuda.set_stream(torch.cuda.Stream(device=dev))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush_rd = torch.ones(64 << 20, dtype=torch.int32, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def per_op(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        flush.zero_()
        flush_rd.max()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def run(name, pat, m, n, k, tp):
    p = fx.ProblemSpec(m, n, k, tp, pat)
    comm = fx.Communicator(tp, [0] * tp, heap_bytes=fx.required_heap_bytes(p) + (64 << 20))
    g = torch.Generator(device=dev).manual_seed(1)
    for r in range(tp):
        for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
            t = comm.tensor(r, kind, p)
            t.copy_(torch.rand(t.shape, device=dev, generator=g).mul_(2).sub_(1))
    s = [torch.cuda.current_stream().cuda_stream] * tp
    tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
    res = {"shape": name, "m": m, "n": n, "k": k, "tp": tp}
    outs = {}
    for label, dk in (("tile", fx.DECODE_TILE), ("stream", fx.DECODE_STREAM)):
        o = fx.default_opts(decode_kernel=dk)
        op = (lambda: comm.ag_gemm(p, tile, m // tp, fx.PULL, True, o, s)) if pat == 0 else \
            (lambda: comm.gemm_rs(p, tile, fx.WRITE_ALLTOALL, True, o, s))
        op()
        comm.sync()
        outs[label] = [comm.tensor(r, N.BUF_C_OUT, p).float().clone() for r in range(tp)]
        res[f"{label}_us"] = per_op(op)
        res[f"{label}_local_us"] = per_op(lambda: comm.local_gemm(p, o, s))
        comm.set_timing(True)
        op()
        comm.sync()
        res[f"{label}_kernel_us"] = comm.last_kernel_ms() * 1e3
        comm.set_timing(False)
    # torch fp32 reference of the same bf16 operands
    a = [comm.tensor(r, N.BUF_A_SHARD, p).float() for r in range(tp)]
    b = [comm.tensor(r, N.BUF_B_SHARD, p).float() for r in range(tp)]
    if pat == 0:
        ag = torch.cat(a, 0)
        want = [ag @ b[r].t() for r in range(tp)]
    else:
        full = sum(a[r] @ b[r].t() for r in range(tp))
        rpr = m // tp
        want = [full[r * rpr:(r + 1) * rpr] for r in range(tp)]
    for label in ("tile", "stream"):
        err = max(((outs[label][r] - want[r]).abs() / want[r].abs().clamp_min(1.0)).max().item() for r in range(tp))
        res[f"{label}_max_rel_err"] = err
    res["stream_vs_tile"] = max((outs["stream"][r] - outs["tile"][r]).abs().max().item() for r in range(tp))
    if tp == 1:
        aa, ww = a[0].bfloat16().contiguous(), b[0].bfloat16().contiguous()
        out = torch.empty(aa.shape[0], ww.shape[0], dtype=torch.bfloat16, device=dev)
        res["cublas_us"] = per_op(lambda: torch.matmul(aa, ww.t(), out=out))
    res["weight_MB"] = sum(x.numel() for x in b) * 2 / 1e6
    res["hbm_roofline_us"] = res["weight_MB"] / 6538.3 * 1e3
    print(json.dumps(res), flush=True)
    comm.close()


for name, spec in SHAPES.items():
    if len(sys.argv) > 1 and name not in sys.argv[1:]:
        continue
    run(name, *spec)
