"""Is the AG overhead generic? Times the plain local GEMM of L-AG (all 8
emulated ranks) alone and with an unrelated 470 MB device-to-device copy (the
volume the emulated AllGather moves) running concurrently on another stream.
Round-robin medians (profiling aid)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N
from bench import WORKLOADS

pattern, m, n, k, tp, _ = WORKLOADS["llama70b-up-ag"]
p = fx.ProblemSpec(m, n, k, tp, pattern)
cs = torch.cuda.Stream()
torch.cuda.set_stream(cs)
comm = fx.Communicator(tp, [0] * tp, heap_bytes=fx.required_heap_bytes(p) + (64 << 20))
for r in range(tp):
    for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD, N.BUF_A_AGG):
        t = comm.tensor(r, kind, p)
        t.copy_(torch.rand(t.shape, device="cuda").mul_(2).sub_(1))
src = torch.empty(470 << 20, dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
side = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = [cs.cuda_stream] * tp
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
times = {"gemm alone": [], "gemm + concurrent 470 MB copy": [], "copy alone": []}
for _ in range(3):
    comm.local_gemm(p, None, st)
torch.cuda.synchronize()
for _ in range(15):
    for name in times:
        flush.zero_()
        torch.cuda.synchronize()
        e0.record(cs)
        if name != "copy alone":
            if "copy" in name:
                side.wait_event(e0)
                with torch.cuda.stream(side):
                    dst.copy_(src)
            comm.local_gemm(p, None, st)
        else:
            dst.copy_(src)
        if "copy" in name and name != "copy alone":
            cs.wait_stream(side)
        e1.record(cs)
        e1.synchronize()
        times[name].append(e0.elapsed_time(e1))
for name, ts in times.items():
    print(f"{name:36s} median {statistics.median(ts) * 1e3:8.1f} us")
