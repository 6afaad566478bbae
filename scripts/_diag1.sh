for nf in "" 1; do
echo "=== C1 RS NOFLUSH=$nf"; NOFLUSH=$nf timeout 120 python scripts/stream_trace.py 1 1024 1024 1024 2 1 2>&1 | grep -v "warp [0-7] at"
done
python - <<'PY'
import torch, paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N
p = fx.ProblemSpec(1024, 1024, 1024, 2, fx.GEMM_REDUCESCATTER)
comm = fx.Communicator(2, [0, 0], heap_bytes=fx.required_heap_bytes(p) + (64 << 20))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); rd = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for name, fn in (("local", lambda: comm.local_gemm(p, None, [s, s])), ("fused", lambda: comm.gemm_rs(p, fx.TileShape(512, 1024), fx.WRITE_ALLTOALL, True, None, [s, s]))):
    comm.set_timing(True)
    ts = []
    for i in range(12):
        flush.zero_(); rd.max()
        fn(); comm.sync(); ts.append(comm.last_kernel_ms() * 1e3)
    print(name, "kernel us", sorted(ts)[6])
a = torch.randn(1024, 512, device="cuda", dtype=torch.bfloat16); b = torch.randn(1024, 512, device="cuda", dtype=torch.bfloat16)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts=[]
for i in range(12):
    flush.zero_(); rd.max(); e0.record(); c = a @ b.t(); c2 = a @ b.t(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1)*1e3)
print("cublas 2x(1024x1024x512) us", sorted(ts)[6])
PY
