"""Achievable HBM bandwidth on this GPU (profiling aid): read-only (sum),
copy (read+write) over 470 MB — the decode sweep's weight volume — with CUDA
events, best of 20."""
import torch

torch.cuda.init()
x = torch.empty(470 * 1024 * 1024 // 2, dtype=torch.bfloat16, device="cuda").uniform_()
y = torch.empty_like(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def best(fn, n=20):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(n):
        e0.record(); fn(); e1.record(); e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out)


nb = x.numel() * 2
t = best(lambda: x.sum(dtype=torch.float32))
print(f"read-only (sum): {nb / t / 1e6:.0f} GB/s  ({t * 1e3:.1f} us for {nb / 1e6:.0f} MB)")
t = best(lambda: y.copy_(x))
print(f"copy: {2 * nb / t / 1e6:.0f} GB/s (read+write bytes)")
