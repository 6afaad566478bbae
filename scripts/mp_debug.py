import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N
from oracle import oracle as O
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
def gather(blob):
    out = [None] * world; dist.all_gather_object(out, blob); return out
pat, m, n, k = fx.GEMM_REDUCESCATTER, 8 * world, 512, 128 * world
p = fx.ProblemSpec(m, n, k, world, pat)
comm = fx.Communicator.ipc(rank, world, 0, fx.required_heap_bytes(p) + (8 << 20), gather)
a_bits, bt_bits = O.rank_inputs_bits(pat, m, n, k, world, 11, rank)
comm.tensor(rank, N.BUF_A_SHARD, p).copy_(torch.from_numpy(a_bits.view(np.int16)).cuda().view(torch.bfloat16))
comm.tensor(rank, N.BUF_B_SHARD, p).copy_(torch.from_numpy(bt_bits.view(np.int16)).cuda().view(torch.bfloat16))
torch.cuda.synchronize(); dist.barrier()
for it in range(3):
    comm.gemm_rs(p, fx.TileShape(p.rows_per_rank(), p.n), fx.WRITE_ALLTOALL, True, fx.default_opts(out_dtype=fx.F32, wall_budget_s=20, trace=1))
    comm.sync()
    got = comm.tensor(rank, N.BUF_C_OUT_F32, p).double().cpu().numpy()
    a_all, b_all = zip(*[O.rank_inputs(pat, m, n, k, world, 11, r, True) for r in range(world)])
    want = O.dense_oracle(pat, m, n, k, world, a_all, b_all)[rank]
    bad = np.argwhere(np.abs(got - want) > 1e-3 * np.maximum(1, np.abs(want)))
    ev = fx.comm.read_trace(comm, rank, p)
    print("DBG", rank, it, "err", O.max_rel_error(got, want), "nbad", len(bad), "rows", sorted(set(bad[:, 0].tolist()))[:10] if len(bad) else [],
          "cols", sorted(set((bad[:, 1] // 256).tolist())) if len(bad) else [], "events", [(e["event"], e["tile_col"], e["target"]) for e in ev], flush=True)
    print("DBG", rank, "got", got[0, :4], "want", want[0, :4], flush=True)
    dist.barrier()
comm.close()
