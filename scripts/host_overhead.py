"""Host-side cost of enqueueing one fused operator (the call returns after the
work is queued): median wall time of the API call, for the headline and the
decode shapes, with the launch profile of each phase if FLUX_HOST_PROFILE=1."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_06858_b200 as fx  # noqa: E402

torch.cuda.set_stream(torch.cuda.Stream())
s = torch.cuda.current_stream().cuda_stream
for name, pat, m, n, k, tp in (("L-AG emulated tp8", 0, 4096, 28672, 8192, 8), ("rank AG m16", 0, 16, 3584, 8192, 1),
                               ("rank RS m16", 1, 16, 8192, 3584, 1), ("decode RS m16 tp8", 1, 16, 8192, 28672, 8)):
    p = fx.ProblemSpec(m, n, k, tp, pat)
    comm = fx.Communicator(tp, [0] * tp, heap_bytes=fx.required_heap_bytes(p) + (16 << 20))
    tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
    opts = fx.default_opts()
    if pat == 0:
        fn = lambda: comm.ag_gemm(p, tile, p.rows_per_rank(), fx.PULL, True, opts, [s] * tp)
    else:
        fn = lambda: comm.gemm_rs(p, tile, fx.WRITE_ALLTOALL, True, opts, [s] * tp)
    for _ in range(3):
        fn()
    comm.sync()
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        comm.sync()
    ts.sort()
    print(f"{name:20s} host enqueue median {ts[10]*1e6:8.1f} us  min {ts[0]*1e6:8.1f} us", flush=True)
    comm.close()
