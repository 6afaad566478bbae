"""Profiling aid: per-CTA phase times of one streaming-kernel launch from the
device trace (kEvLaunch tile_col 0 = CTA start, 2 = producer issued its last
load, 3 = a segment's accumulator drained, 1 = CTA end).

    python scripts/stream_trace.py [pattern m n k tp]
"""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2406_06858_b200 as fx  # noqa: E402
from paper_2406_06858_b200 import _native as N  # noqa: E402
from paper_2406_06858_b200.comm import read_trace  # noqa: E402

pat, m, n, k, tp = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (0, 16, 3584, 8192, 1)))
dk = int(sys.argv[6]) if len(sys.argv) > 6 else fx.DECODE_STREAM
p = fx.ProblemSpec(m, n, k, tp, pat)
torch.cuda.set_stream(torch.cuda.Stream())
comm = fx.Communicator(tp, [0] * tp, heap_bytes=fx.required_heap_bytes(p) + (64 << 20))
for r in range(tp):
    for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
        t = comm.tensor(r, kind, p)
        t.copy_(torch.rand(t.shape, device="cuda").mul_(2).sub_(1))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
s = [torch.cuda.current_stream().cuda_stream] * tp
tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
for trace in (0, 0, 0, 1):
    o = fx.default_opts(trace=trace, decode_kernel=dk)
    if not os.environ.get("NOFLUSH"):
        flush.zero_()
        flush_rd.max()
    comm.set_timing(True)
    if pat == 0:
        comm.ag_gemm(p, tile, m // tp, fx.PULL, True, o, s)
    else:
        comm.gemm_rs(p, tile, fx.WRITE_ALLTOALL, True, o, s)
    comm.sync()
    print(f"trace={trace} kernel {comm.last_kernel_ms() * 1e3:.1f} us")
allev = read_trace(comm, 0, p)
t0 = min(e["ts"] for e in allev)
by = {}
for e in allev:
    key = ("launch", e["tile_col"]) if e["event"] == "launch" else (e["event"], None)
    by.setdefault(key, []).append((e["ts"] - t0) / 1e3)
names = {0: "cta start", 2: "producer done", 3: "segment drained", 4: "split wait done", 5: "split share done",
         1: "cta end", 10: "AG piece loaded", 11: "AG stores done", 12: "AG transfer start", 13: "RS unit summed", 14: "RS unit bar (t0)", 15: "RS unit bar (t32)", 20: "RS group w2-3 done",
         21: "RS group epi done", 22: "RS group w0-1 done", 6: "epi segs drained", 7: "epi splits done", 8: "w0-1 join RS",
         **{24 + w: f"warp {w} at exit" for w in range(8)},
         30: "prologue done", 32: "first stage landed", 33: "first acc ready", 34: "first tile stored",
         35: "1st tile chunk 1", 38: "1st tile chunk 4"}
for key in sorted(by, key=lambda k: sorted(by[k])[len(by[k]) // 2]):
    v = sorted(by[key])
    name = names.get(key[1], key[0]) if key[0] == "launch" else key[0]
    print(f"{name:>16s}: n={len(v):4d} min {v[0]:7.2f}  p10 {v[len(v) // 10]:7.2f}  med {v[len(v) // 2]:7.2f}  "
          f"p90 {v[9 * len(v) // 10]:7.2f}  max {v[-1]:7.2f} us")
