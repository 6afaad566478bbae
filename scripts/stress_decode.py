"""Randomised stress of the decode paths (streaming kernel: stream-K, whole
tiles, cluster split-K in buffer and ring mode; the emulated NVLS protocol)
against the CPU oracle: random token counts, widths, depths, TP degrees and
interleaving jitter; prints one line per failure and a summary.

    python scripts/stress_decode.py [seconds] [seed] [tile]
("tile": medium shapes on the tile kernel with random CTA grouping, transfer
engine and partial precision instead)."""
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401

import paper_2406_06858_b200 as fx  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import gpu_harness as H  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
tile_mode = len(sys.argv) > 3 and sys.argv[3] == "tile"  # medium shapes on the tile kernel, every knob
t_end = time.time() + budget
runs = fails = 0
while time.time() < t_end:
    pat = rng.choice([fx.ALLGATHER_GEMM, fx.GEMM_REDUCESCATTER])
    tp = rng.choice([1, 1, 2, 4, 8])
    m = tp * rng.randint(1, max(1, 64 // tp))
    extra = {}
    if tile_mode:
        tp = rng.choice([1, 2, 3, 4, 8])
        m = tp * rng.choice([16, 64, 128, 200, 256, 384, 512])
    if pat == fx.ALLGATHER_GEMM:
        n = tp * 8 * rng.randint(1, 64)
        k = 64 * rng.randint(1, 48)
    else:
        n = 8 * rng.randint(1, 160)
        k = tp * 64 * rng.randint(1, 24)
    nvls = rng.choice([0, 0, 2]) if tp > 1 else 0
    if tile_mode:
        extra = dict(decode_kernel=fx.DECODE_TILE, cta_group=rng.choice([0, 1, 2]),
                     ag_engine=rng.choice([0, 1, 2]) if nvls == 0 else 0)
        if pat == fx.GEMM_REDUCESCATTER and nvls == 0 and rng.random() < 0.25:
            extra["rs_partials"] = fx.BF16
    seed = rng.randint(0, 1 << 30)
    jitter = rng.choice([0, 0, seed])
    p = fx.ProblemSpec(m, n, k, tp, pat)
    try:
        with H.make_comm(p) as comm:
            a, b = H.upload(comm, p, seed=seed % 1000)
            kw = dict(decode_kernel=fx.DECODE_STREAM)
            kw.update(extra)
            opts = fx.default_opts(out_dtype=fx.F32, wall_budget_s=10.0, nvls=nvls, interleave_seed=jitter, **kw)
            tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
            for _ in range(2):
                if pat == fx.ALLGATHER_GEMM:
                    comm.ag_gemm(p, tile, 0, fx.PULL, True, opts)
                else:
                    comm.gemm_rs(p, tile, fx.WRITE_ALLTOALL, True, opts)
            comm.sync()
            got = H.outputs(comm, p, True)
            want = O.dense_oracle(pat, m, n, k, tp, a, b)
            if "rs_partials" in extra:  # bf16 partials: checked normwise
                err = max(O.normwise_error(g, w) for g, w in zip(got, want))
                tol = 5e-3
            else:
                err = max(O.max_rel_error(g, w) for g, w in zip(got, want))
                tol = H.tol(True, k)
            if not err <= tol:
                fails += 1
                print(f"FAIL pat={pat} m={m} n={n} k={k} tp={tp} nvls={nvls} jitter={jitter} {extra}: err {err:.3e}", flush=True)
    except fx.FluxError as e:
        fails += 1
        print(f"ERROR pat={pat} m={m} n={n} k={k} tp={tp} nvls={nvls} {extra}: {e}", flush=True)
    runs += 1
print(f"STRESS runs={runs} failures={fails}", flush=True)
