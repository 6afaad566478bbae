"""First GPU probe: plain GEMM vs torch, AG / RS emulated on one GPU."""
import sys, time, torch
sys.path.insert(0, ".")
import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N

torch.manual_seed(0)

def rel(a, b):
    a = a.double(); b = b.double()
    return ((a - b).abs() / torch.clamp(torch.maximum(a.abs(), b.abs()), min=1.0)).max().item()

def fill(comm, r, kind, prob, t):
    v = comm.tensor(r, kind, prob)
    v.copy_(t)

for (m, n, k) in [(128, 256, 64), (256, 512, 128), (1024, 1024, 1024), (300, 200, 100)]:
    prob = fx.ProblemSpec(m, n, k, 1, fx.ALLGATHER_GEMM)
    with fx.Communicator(1, [0], heap_bytes=fx.required_heap_bytes(prob)) as comm:
        A = torch.rand(m, k, device="cuda").mul(2).sub(1).bfloat16()
        B = torch.rand(n, k, device="cuda").mul(2).sub(1).bfloat16()
        fill(comm, 0, N.BUF_A_AGG, prob, A)
        fill(comm, 0, N.BUF_B_SHARD, prob, B)
        torch.cuda.synchronize()
        comm.local_gemm(prob, fx.default_opts(out_dtype=fx.F32))
        comm.sync()
        C = comm.tensor(0, N.BUF_C_OUT_F32, prob).clone()
        ref = A.float() @ B.float().t()
        print("plain", m, n, k, "rel", rel(C, ref), flush=True)

# timing plain GEMM 8192^3
m = n = k = 8192
prob = fx.ProblemSpec(m, n, k, 1, fx.ALLGATHER_GEMM)
with fx.Communicator(1, [0], heap_bytes=fx.required_heap_bytes(prob)) as comm:
    A = torch.randn(m, k, device="cuda").bfloat16(); B = torch.randn(n, k, device="cuda").bfloat16()
    fill(comm, 0, N.BUF_A_AGG, prob, A); fill(comm, 0, N.BUF_B_SHARD, prob, B)
    for _ in range(3): comm.local_gemm(prob)
    comm.sync()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    st = torch.cuda.current_stream().cuda_stream
    s.record(); 
    for _ in range(10): comm.local_gemm(prob, streams=[st])
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print("plain 8192^3 ms", ms, "TFLOPS", 2 * m * n * k / ms / 1e9, flush=True)
    C = comm.tensor(0, N.BUF_C_OUT, prob)
    ref = (A[:256].float() @ B.float().t())
    print("plain 8192 rel(first 256 rows)", rel(C[:256].float(), ref))
    s.record()
    for _ in range(10): torch.matmul(A, B.t())
    e.record(); torch.cuda.synchronize(); ms = s.elapsed_time(e) / 10
    print("torch 8192^3 ms", ms, "TFLOPS", 2 * m * n * k / ms / 1e9, flush=True)

# AG emulated TP=4
for (m, n, k, tp, rpct) in [(512, 1024, 256, 4, 128), (1024, 2048, 512, 4, 64), (16, 16, 16, 4, 4)]:
    prob = fx.ProblemSpec(m, n, k, tp, fx.ALLGATHER_GEMM)
    with fx.Communicator(tp, [0] * tp, heap_bytes=fx.required_heap_bytes(prob)) as comm:
        As = [torch.rand(m // tp, k, device="cuda").mul(2).sub(1).bfloat16() for _ in range(tp)]
        Bs = [torch.rand(n // tp, k, device="cuda").mul(2).sub(1).bfloat16() for _ in range(tp)]
        for r in range(tp):
            fill(comm, r, N.BUF_A_SHARD, prob, As[r]); fill(comm, r, N.BUF_B_SHARD, prob, Bs[r])
        torch.cuda.synchronize()
        comm.ag_gemm(prob, fx.TileShape(m // tp, n // tp), rpct, fx.PULL, True, fx.default_opts(out_dtype=fx.F32, wall_budget_s=5.0))
        comm.sync()
        Ag = torch.cat(As).float()
        worst = max(rel(comm.tensor(r, N.BUF_C_OUT_F32, prob), Ag @ Bs[r].float().t()) for r in range(tp))
        print("AG", m, n, k, tp, rpct, "rel", worst, flush=True)

# RS emulated
for (m, n, k, tp) in [(1024, 512, 256, 4), (512, 512, 1024, 2), (16, 16, 16, 4), (2048, 1024, 512, 8)]:
    prob = fx.ProblemSpec(m, n, k, tp, fx.GEMM_REDUCESCATTER)
    with fx.Communicator(tp, [0] * tp, heap_bytes=fx.required_heap_bytes(prob)) as comm:
        As = [torch.rand(m, k // tp, device="cuda").mul(2).sub(1).bfloat16() for _ in range(tp)]
        Bs = [torch.rand(n, k // tp, device="cuda").mul(2).sub(1).bfloat16() for _ in range(tp)]
        for r in range(tp):
            fill(comm, r, N.BUF_A_SHARD, prob, As[r]); fill(comm, r, N.BUF_B_SHARD, prob, Bs[r])
        torch.cuda.synchronize()
        for it in range(3):
            comm.gemm_rs(prob, fx.TileShape(m // tp, n), fx.WRITE_ALLTOALL, True, fx.default_opts(out_dtype=fx.F32, wall_budget_s=5.0))
            comm.sync()
        full = sum(As[r].float() @ Bs[r].float().t() for r in range(tp))
        rpr = m // tp
        worst = max(rel(comm.tensor(r, N.BUF_C_OUT_F32, prob), full[r * rpr:(r + 1) * rpr]) for r in range(tp))
        print("RS", m, n, k, tp, "rel", worst, flush=True)
        comm.nonoverlap(prob, fx.default_opts(out_dtype=fx.F32)); comm.sync()
        worst = max(rel(comm.tensor(r, N.BUF_C_OUT_F32, prob), full[r * rpr:(r + 1) * rpr]) for r in range(tp))
        print("RS nonoverlap", m, n, k, tp, "rel", worst, flush=True)
print("DONE")
