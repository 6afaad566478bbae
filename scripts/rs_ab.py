"""Profiling aid: per-op device time of decode GEMM-RS / AG-GEMM shapes (ranks
emulated on one GPU, L2 flushed between ops) for the package under ROOT
(A/B of two builds: two package roots, or one root and FLUX_LIB_PATH).
python scripts/rs_ab.py ROOT [shape ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, sys.argv[1])
import paper_2406_06858_b200 as fx  # noqa: E402
from paper_2406_06858_b200 import _native as N  # noqa: E402

SHAPES = {"rs-down-m16-tp8": (1, 16, 8192, 28672, 8), "rs-attn-m16-tp8": (1, 16, 8192, 8192, 8),
          "rs-down-m128-tp8": (1, 128, 8192, 28672, 8), "rs-attn-m128-tp8": (1, 128, 8192, 8192, 8),
          "ag-up-m128-tp8": (0, 128, 28672, 8192, 8), "rs-1024-tp2": (1, 1024, 1024, 1024, 2),
          "ag-up-m16-tp8": (0, 16, 28672, 8192, 8), "ag-up-m512-tp8": (0, 512, 28672, 8192, 8),
          # one GPU's TP=8 decode share (tp=1 problems with the per-rank shapes)
          "rank-rs-attn-m128": (1, 128, 8192, 1024, 1), "rank-rs-attn-m512": (1, 512, 8192, 1024, 1),
          "rank-rs-down-m128": (1, 128, 8192, 3584, 1), "rank-rs-down-m512": (1, 512, 8192, 3584, 1),
          "rs-attn-m512-tp8": (1, 512, 8192, 8192, 8),
          "rank-rs-attn-m16": (1, 16, 8192, 1024, 1), "rank-rs-attn-m64": (1, 64, 8192, 1024, 1),
          "rank-rs-down-m16": (1, 16, 8192, 3584, 1), "rank-rs-down-m64": (1, 64, 8192, 3584, 1),
          "rank-ag-up-m128": (0, 128, 3584, 8192, 1), "rank-ag-up-m64": (0, 64, 3584, 8192, 1),
          "rank-ag-up-m32": (0, 32, 3584, 8192, 1), "rank-ag-up-m16": (0, 16, 3584, 8192, 1),
          "rank-ag-up-m256": (0, 256, 3584, 8192, 1), "rank-ag-up-m192": (0, 192, 3584, 8192, 1)}
if len(sys.argv) > 2:
    SHAPES = {k: v for k, v in SHAPES.items() if k in sys.argv[2:]}
dev = torch.device("cuda", 0)
torch.cuda.set_stream(torch.cuda.Stream(device=dev))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush_rd = torch.ones(64 << 20, dtype=torch.int32, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, (pat, m, n, k, tp) in SHAPES.items():
    p = fx.ProblemSpec(m, n, k, tp, pat)
    comm = fx.Communicator(tp, [0] * tp, heap_bytes=fx.required_heap_bytes(p) + (64 << 20))
    for r in range(tp):
        for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
            t = comm.tensor(r, kind, p)
            t.copy_(torch.rand(t.shape, device=dev).mul_(2).sub_(1))
    s = [torch.cuda.current_stream().cuda_stream] * tp
    tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
    o = fx.default_opts()
    if hasattr(o, "decode_kernel"):
        o.decode_kernel = int(os.environ.get("DK", "1"))  # 1 = tile kernel (default here), 0 = auto, 2 = streaming
    op = (lambda: comm.ag_gemm(p, tile, m // tp, fx.PULL, True, o, s)) if pat == 0 else \
        (lambda: comm.gemm_rs(p, tile, fx.WRITE_ALLTOALL, True, o, s))
    for _ in range(3):
        op()
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        flush.zero_()
        flush_rd.max()
        e0.record()
        op()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(json.dumps({"root": sys.argv[1], "lib": os.environ.get("FLUX_LIB_PATH", ""), "shape": name, "us": round(ts[len(ts) // 2], 1)}), flush=True)
    comm.close()
