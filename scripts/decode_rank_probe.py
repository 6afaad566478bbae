"""Profiling aid: one GPU's decode share (the rank-decode-* bench workloads) —
per-op time with the bench's L2 flush between ops vs back-to-back ops, our
kernel vs cuBLAS, to separate the kernel's streaming rate from fixed costs."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2406_06858_b200 as fx  # noqa: E402
from paper_2406_06858_b200 import _native as N  # noqa: E402

SHAPES = {
    "ag-up-m16": (0, 16, 3584, 8192), "rs-down-m16": (1, 16, 8192, 3584), "rs-attn-m16": (1, 16, 8192, 1024),
    "ag-up-m128": (0, 128, 3584, 8192), "rs-down-m128": (1, 128, 8192, 3584),
}
dev = torch.device("cuda", 0)
torch.cuda.set_stream(torch.cuda.Stream(device=dev))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush_rd = torch.ones(64 << 20, dtype=torch.int32, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def per_op(fn, n=20, flushed=True):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        if flushed:
            flush.zero_()
            flush_rd.max()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def burst(fn, n=50):
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


for name, (pat, m, n, k) in SHAPES.items():
    if len(sys.argv) > 1 and name not in sys.argv[1:]:
        continue
    p = fx.ProblemSpec(m, n, k, 1, pat)
    comm = fx.Communicator(1, [0], heap_bytes=fx.required_heap_bytes(p) + (64 << 20))
    for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
        t = comm.tensor(0, kind, p)
        t.copy_(torch.rand(t.shape, device=dev).mul_(2).sub_(1))
    s = [torch.cuda.current_stream().cuda_stream]
    tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
    op = (lambda: comm.ag_gemm(p, tile, m, fx.PULL, True, None, s)) if pat == 0 else \
        (lambda: comm.gemm_rs(p, tile, fx.WRITE_ALLTOALL, True, None, s))
    local = lambda: comm.local_gemm(p, None, s)  # noqa: E731
    a = comm.tensor(0, N.BUF_A_SHARD, p).contiguous()
    w = comm.tensor(0, N.BUF_B_SHARD, p).contiguous()
    out = torch.empty(a.shape[0], w.shape[0], dtype=torch.bfloat16, device=dev)
    cub = lambda: torch.matmul(a, w.t(), out=out)  # noqa: E731
    wbytes = w.numel() * 2
    comm.set_timing(True)
    op()
    comm.sync()
    kern = comm.last_kernel_ms() * 1e3
    comm.set_timing(False)
    row = {"shape": name, "weight_MB": wbytes / 1e6, "hbm_roofline_us": wbytes / 6535e3,
           "op_flushed_us": per_op(op), "op_burst_us": burst(op), "op_kernel_us_lib_events": kern,
           "local_flushed_us": per_op(local), "local_burst_us": burst(local),
           "cublas_flushed_us": per_op(cub), "cublas_burst_us": burst(cub)}
    print(row, flush=True)
    comm.close()
