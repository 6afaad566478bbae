"""Small fused runs for compute-sanitizer (memcheck / racecheck / synccheck):
AG on both transfer engines, RS chained / owner-sum / decode owner units,
FusedReduce, the dynamic tile scheduler, the streaming decode kernel (cluster
split-K in buffer and ring mode, stream-K), the emulated NVLS protocol,
and the MLP chain, each checked against a cuBLAS product. Usage:
    compute-sanitizer --tool memcheck python scripts/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N


def fill(comm, p, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    for r in range(p.tp):
        for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
            t = comm.tensor(r, kind, p)
            t.copy_((torch.rand(t.shape, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16))


def check(comm, p, tag, bf16_partials=False):
    a = [comm.tensor(r, N.BUF_A_SHARD, p).float() for r in range(p.tp)]
    b = [comm.tensor(r, N.BUF_B_SHARD, p).float() for r in range(p.tp)]
    worst = 0.0
    for r in range(p.tp):
        got = comm.tensor(r, N.BUF_C_OUT, p).float()
        if p.pattern == fx.ALLGATHER_GEMM:
            ref = torch.cat(a) @ b[r].t()
        else:
            rpr = p.rows_per_rank()
            ref = sum(a[s][r * rpr:(r + 1) * rpr] @ b[s].t() for s in range(p.tp))
        worst = max(worst, ((got - ref).abs().max() / ref.abs().max().clamp(min=1)).item())
    print(f"{tag}: max err {worst:.2e}", flush=True)
    assert worst < (3e-2 if bf16_partials else 1e-2), tag


cases = [("AG copy engines", fx.ProblemSpec(512, 1024, 256, 4, fx.ALLGATHER_GEMM), dict(ag_engine=1)),
         ("AG in-kernel", fx.ProblemSpec(512, 1024, 256, 4, fx.ALLGATHER_GEMM), dict(ag_engine=2)),
         ("RS chained (aligned blocks, long sections)", fx.ProblemSpec(4096, 4096, 512, 4, fx.GEMM_REDUCESCATTER), {}),
         ("AG tail split (K-slices)", fx.ProblemSpec(1024, 2048, 512, 8, fx.ALLGATHER_GEMM), dict(ag_engine=1)),
         ("RS owner sum (Naive swizzle)", fx.ProblemSpec(1024, 512, 512, 4, fx.GEMM_REDUCESCATTER), {}),
         ("RS decode (owner reduction units)", fx.ProblemSpec(64, 512, 512, 4, fx.GEMM_REDUCESCATTER), {}),
         ("RS decode, blocks straddling tiles", fx.ProblemSpec(360, 515, 96, 8, fx.GEMM_REDUCESCATTER), {}),
         ("AG dynamic scheduler", fx.ProblemSpec(1024, 2048, 512, 8, fx.ALLGATHER_GEMM), dict(env="FLUX_DYN_SCHED")),
         ("RS dynamic scheduler", fx.ProblemSpec(4096, 4096, 512, 4, fx.GEMM_REDUCESCATTER), dict(env="FLUX_DYN_SCHED")),
         ("RS FusedReduce", fx.ProblemSpec(1024, 512, 512, 4, fx.GEMM_REDUCESCATTER), dict(deterministic_reduce=0)),
         ("AG in-kernel Push", fx.ProblemSpec(512, 1024, 256, 4, fx.ALLGATHER_GEMM), dict(ag_engine=2, push=1)),
         ("RS smaller than a wave (owner units)", fx.ProblemSpec(1024, 1024, 512, 2, fx.GEMM_REDUCESCATTER), {}),
         ("RS decode, bf16 partials", fx.ProblemSpec(64, 512, 512, 4, fx.GEMM_REDUCESCATTER), dict(rs_partials=fx.BF16)),
         ("AG graph-safe", fx.ProblemSpec(512, 1024, 256, 4, fx.ALLGATHER_GEMM), dict(graph_safe=1)),
         # streaming decode kernel: cluster split-K (buffer / ring mode), stream-K, whole tiles
         ("stream AG, clusters of 8", fx.ProblemSpec(16, 1024, 2048, 1, fx.ALLGATHER_GEMM), dict(decode_kernel=2)),
         ("stream RS M=64, cluster ring mode", fx.ProblemSpec(64, 1024, 2048, 1, fx.GEMM_REDUCESCATTER),
          dict(decode_kernel=2)),
         ("stream RS tp=4, clusters", fx.ProblemSpec(16, 1024, 1024, 4, fx.GEMM_REDUCESCATTER), dict(decode_kernel=2)),
         ("stream AG stream-K segments", fx.ProblemSpec(16, 1024, 8192, 1, fx.ALLGATHER_GEMM),
          dict(decode_kernel=2, env="FLUX_SK_CLUSTER")),
         # NVLS protocol (emulated multicast)
         ("NVLS AG (emulated)", fx.ProblemSpec(512, 1024, 256, 4, fx.ALLGATHER_GEMM), dict(nvls=2)),
         ("NVLS RS units (emulated)", fx.ProblemSpec(512, 1024, 512, 4, fx.GEMM_REDUCESCATTER), dict(nvls=2)),
         ("NVLS RS stream (emulated)", fx.ProblemSpec(16, 1024, 1024, 4, fx.GEMM_REDUCESCATTER), dict(nvls=2, decode_kernel=2))]
only = os.environ.get("SANITIZE_ONLY")  # e.g. "0,1": run these case indices
if only:
    cases = [cases[int(i)] for i in only.split(",")]
for tag, p, kw in cases:
    kw = dict(kw)
    env = kw.pop("env", None)
    push = kw.pop("push", 0)
    for var in ("FLUX_DYN_SCHED", "FLUX_SK_CLUSTER"):
        os.environ.pop(var, None)
    if env:
        os.environ[env] = "1"
    with fx.Communicator(p.tp, [0] * p.tp, heap_bytes=fx.required_heap_bytes(p)) as comm:
        fill(comm, p, 1)
        opts = fx.default_opts(wall_budget_s=120.0, **kw)
        tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
        if p.pattern == fx.ALLGATHER_GEMM:
            comm.ag_gemm(p, tile, p.rows_per_rank(), fx.PUSH if push else fx.PULL, True, opts)
        else:
            wm = fx.FUSED_REDUCE if kw.get("deterministic_reduce") == 0 else fx.WRITE_ALLTOALL
            comm.gemm_rs(p, tile, wm, "Naive" not in tag, opts)
        comm.sync()
        check(comm, p, tag, kw.get("rs_partials") == fx.BF16)
if only:
    print("SANITIZE-RUN-DONE", flush=True)
    sys.exit(0)
spec = fx.MlpSpec(m=512, hidden=256, ffn=1024, tp=2, activation=fx.ACT_GELU)
x = [torch.randn(256, 256, device="cuda").to(torch.bfloat16) for _ in range(2)]
wu = [torch.randn(512, 256, device="cuda").mul(0.05).to(torch.bfloat16) for _ in range(2)]
wd = [torch.randn(256, 512, device="cuda").mul(0.05).to(torch.bfloat16) for _ in range(2)]
act = [torch.empty(512, 512, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
out = [torch.empty(256, 256, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
with fx.Communicator(2, [0, 0], heap_bytes=spec.required_heap_bytes()) as comm:
    comm.mlp_forward(spec, [dict(x=x[r], w_up=wu[r], w_down=wd[r], act=act[r], out=out[r]) for r in range(2)],
                     opts=fx.default_opts(wall_budget_s=120.0))
    comm.sync()
print("MLP chain: ok")
print("SANITIZE-RUN-DONE")
