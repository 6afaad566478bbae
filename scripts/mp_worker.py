"""One rank of a multi-process (one process per rank) run of the fused
operators through the IPC communicator. Launched by tests/test_multiprocess_gpu.py
with torchrun; every rank may share one physical GPU (handles are exchanged
over gloo, so no NCCL is needed)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N
from oracle import oracle as O
from oracle import gpu_harness as H

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
ndev = torch.cuda.device_count()
dev = rank % ndev
torch.cuda.set_device(dev)
dist.init_process_group("gloo")


def gather(blob):
    out = [None] * world
    dist.all_gather_object(out, blob)
    return out


results = {}
# (pattern, m, n, k, variant): AG variant = engine (0 auto, 1 copy engines, 2 in-kernel, 3 copy-engine Push,
# 4 in-kernel Push);
# RS variant = 0 WriteAlltoAll, 1 FusedReduce (arrival order), 2 WriteAlltoAll with bf16 partials
cases = [(fx.ALLGATHER_GEMM, 256 * world, 512 * world, 384, 1), (fx.ALLGATHER_GEMM, 256 * world, 512 * world, 384, 2),
         (fx.ALLGATHER_GEMM, 16 * world, 256 * world, 1024, 0), (fx.GEMM_REDUCESCATTER, 512 * world, 768, 256 * world, 0),
         (fx.ALLGATHER_GEMM, 256 * world, 512 * world, 384, 3), (fx.GEMM_REDUCESCATTER, 512 * world, 768, 256 * world, 1),
         (fx.GEMM_REDUCESCATTER, 512 * world, 768, 256 * world, 2),
         (fx.GEMM_REDUCESCATTER, 40 * world, 300, 64 * world, 0),  # decode-sized blocks: owner reduction units
         (fx.ALLGATHER_GEMM, 256 * world, 512 * world, 384, 4)]  # in-kernel Push into the peers' a_agg
heap = max(fx.required_heap_bytes(fx.ProblemSpec(m, n, k, world, pat)) for pat, m, n, k, _ in cases) + (8 << 20)
comm = fx.Communicator.ipc(rank, world, dev, heap, gather)
for pat, m, n, k, engine in cases:
    p = fx.ProblemSpec(m, n, k, world, pat)
    a_bits, bt_bits = O.rank_inputs_bits(pat, m, n, k, world, 7, rank)
    comm.tensor(rank, N.BUF_A_SHARD, p).copy_(torch.from_numpy(a_bits.view(np.int16)).cuda().view(torch.bfloat16))
    comm.tensor(rank, N.BUF_B_SHARD, p).copy_(torch.from_numpy(bt_bits.view(np.int16)).cuda().view(torch.bfloat16))
    torch.cuda.synchronize()
    dist.barrier()
    ag = pat == fx.ALLGATHER_GEMM
    opts = fx.default_opts(out_dtype=fx.F32, wall_budget_s=20.0,
                           ag_engine={3: 1, 4: 2}.get(engine, engine) if ag else 0,
                           deterministic_reduce=0 if (not ag and engine == 1) else 1,
                           rs_partials=fx.BF16 if (not ag and engine == 2) else fx.F32)
    for it in range(3):
        if ag:
            comm.ag_gemm(p, fx.TileShape(p.rows_per_rank(), p.local_cols()), 0, fx.PUSH if engine >= 3 else fx.PULL,
                         True, opts)
        else:
            comm.gemm_rs(p, fx.TileShape(p.rows_per_rank(), p.local_cols()),
                         fx.FUSED_REDUCE if engine == 1 else fx.WRITE_ALLTOALL, True, opts)
    comm.sync()
    got = comm.tensor(rank, N.BUF_C_OUT_F32, p).double().cpu().numpy()
    a_all, b_all = zip(*[O.rank_inputs(pat, m, n, k, world, 7, r, True) for r in range(world)])
    want = O.dense_oracle(pat, m, n, k, world, a_all, b_all)[rank]
    if not ag and engine == 2:  # bf16 partials: normwise
        results[f"{pat}-{m}-{n}-{k}-e{engine}"] = (float(np.linalg.norm(got - want) / np.linalg.norm(want)), 5e-3)
    else:
        results[f"{pat}-{m}-{n}-{k}-e{engine}"] = (O.max_rel_error(got, want), H.tol(True, k))
    dist.barrier()
# The PyTorch custom ops on caller-owned tensors (torch.ops.flux_b200.*).
from paper_2406_06858_b200 import torch_ops  # noqa: E402

cid = torch_ops.register(comm)
for pat, m, n, k in [(fx.ALLGATHER_GEMM, 256 * world, 512 * world, 384), (fx.GEMM_REDUCESCATTER, 256 * world, 512, 128 * world),
                     (fx.GEMM_REDUCESCATTER, 8 * world, 512, 128 * world)]:
    a_bits, bt_bits = O.rank_inputs_bits(pat, m, n, k, world, 11, rank)
    x = torch.from_numpy(a_bits.view(np.int16)).cuda().view(torch.bfloat16)
    w = torch.from_numpy(bt_bits.view(np.int16)).cuda().view(torch.bfloat16)
    dist.barrier()
    out = (torch.ops.flux_b200.ag_gemm(x, w, cid) if pat == fx.ALLGATHER_GEMM
           else torch.ops.flux_b200.gemm_rs(x, w, cid))
    torch.cuda.synchronize()
    a_all, b_all = zip(*[O.rank_inputs(pat, m, n, k, world, 11, r, True) for r in range(world)])
    want = O.dense_oracle(pat, m, n, k, world, a_all, b_all)[rank]
    results[f"torchop-{pat}-{m}-{n}-{k}"] = (O.max_rel_error(out.double().cpu().numpy(), want), H.tol(False, k))
    dist.barrier()
# The chained MLP as an autograd module (torch_ops.TPMlp) against fp32 autograd
# of the same sequence-parallel MLP on the same bf16 values (normwise error).
M, HID, FFN = 256 * world, 256, 512 * world
mlp_heap = max(fx.MlpSpec(M, HID, FFN, world, a).required_heap_bytes() for a in (fx.ACT_GELU, fx.ACT_SWIGLU))
assert mlp_heap <= heap, (mlp_heap, heap)


def _rand(shape, seed, scale=1.0):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return ((torch.rand(shape, generator=g, device="cuda") * 2 - 1) * scale).to(torch.bfloat16)


xs = [_rand((M // world, HID), 100 + r) for r in range(world)]
wus = [_rand((FFN // world, HID), 200 + r, 0.1) for r in range(world)]
wds = [_rand((HID, FFN // world), 300 + r, 0.1) for r in range(world)]
douts = [_rand((M // world, HID), 400 + r) for r in range(world)]
mod = torch_ops.TPMlp(HID, FFN, cid, fx.ACT_GELU, device="cuda")
with torch.no_grad():
    mod.w_up.copy_(wus[rank])
    mod.w_down.copy_(wds[rank])
x = xs[rank].clone().requires_grad_(True)
dist.barrier()
y = mod(x)
y.backward(douts[rank])
torch.cuda.synchronize()
xr = torch.cat(xs).float().requires_grad_(True)
wur = [w.float().requires_grad_(True) for w in wus]
wdr = [w.float().requires_grad_(True) for w in wds]
yr = sum(torch.nn.functional.gelu(xr @ wur[r].t()) @ wdr[r].t() for r in range(world))
yr.backward(torch.cat(douts).float())
rpr = M // world


def _nerr(got, ref):
    return ((got.float() - ref).abs().max() / ref.abs().max().clamp(min=1.0)).item()


results["mlp-out"] = (_nerr(y, yr[rank * rpr:(rank + 1) * rpr].detach()), 3e-2)
results["mlp-dx"] = (_nerr(x.grad, xr.grad[rank * rpr:(rank + 1) * rpr]), 3e-2)
results["mlp-dw_up"] = (_nerr(mod.w_up.grad, wur[rank].grad), 3e-2)
results["mlp-dw_down"] = (_nerr(mod.w_down.grad, wdr[rank].grad), 3e-2)
# The gated variant (SwiGLU, Llama MLP): w_up holds 128 gate + 128 up rows per group.
wus2 = [_rand((2 * FFN // world, HID), 500 + r, 0.1) for r in range(world)]
mod2 = torch_ops.TPMlp(HID, FFN, cid, fx.ACT_SWIGLU, device="cuda")
with torch.no_grad():
    mod2.w_up.copy_(wus2[rank])
    mod2.w_down.copy_(wds[rank])
x2 = xs[rank].clone().requires_grad_(True)
dist.barrier()
y2 = mod2(x2)
y2.backward(douts[rank])
torch.cuda.synchronize()


def _glu(y):
    y4 = y.view(y.shape[0], -1, 2, 128)
    return (torch.nn.functional.silu(y4[:, :, 0]) * y4[:, :, 1]).reshape(y.shape[0], -1)


xr2 = torch.cat(xs).float().requires_grad_(True)
wur2 = [w.float().requires_grad_(True) for w in wus2]
wdr2 = [w.float().requires_grad_(True) for w in wds]
yr2 = sum(_glu(xr2 @ wur2[r].t()) @ wdr2[r].t() for r in range(world))
yr2.backward(torch.cat(douts).float())
results["swiglu-out"] = (_nerr(y2, yr2[rank * rpr:(rank + 1) * rpr].detach()), 3e-2)
results["swiglu-dx"] = (_nerr(x2.grad, xr2.grad[rank * rpr:(rank + 1) * rpr]), 3e-2)
results["swiglu-dw_up"] = (_nerr(mod2.w_up.grad, wur2[rank].grad), 3e-2)
results["swiglu-dw_down"] = (_nerr(mod2.w_down.grad, wdr2[rank].grad), 3e-2)
dist.barrier()
comm.close()
for turn in range(world):  # one rank at a time: the two lines must not interleave on the shared stdout
    if turn == rank:
        sys.stdout.write("RESULT %d %s\n" % (rank, json.dumps(results)))
        sys.stdout.flush()
    dist.barrier()
dist.destroy_process_group()
