"""Parity of the sm_100a fused operators with the CPU oracle, through the C ABI.

Every case runs the real kernels (tcgen05 + TMA GEMM, copy-engine transfer
loop, epilogue P2P partial stores) with all `tp` ranks emulated on cuda:0 —
the reference's threads-as-ranks model (engine.cpp:172-191) on one device.
Tolerance (BASELINE.md parity contract): bf16 inputs, fp32 accumulate and
fp32 cross-rank partials; max_rel_error <= 8e-3 for bf16 outputs and
<= 1e-4·max(1, k/1024) for fp32 outputs (tensor-core accumulation error grows with k; see oracle/gpu_harness.tol).
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_2406_06858_b200 as fx  # noqa: E402
from paper_2406_06858_b200 import _native as N  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import gpu_harness as H  # noqa: E402

AG, RS = fx.ALLGATHER_GEMM, fx.GEMM_REDUCESCATTER
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_ref.json")


def _unhex(rows):
    return np.array([[float.fromhex(v) for v in row] for row in rows], np.float64)


def _run(comm, p, f32=True, transfer=fx.PULL, swizzle=True, rpct=0, write_mode=fx.WRITE_ALLTOALL, **kw):
    opts = fx.default_opts(out_dtype=fx.F32 if f32 else fx.BF16, wall_budget_s=5.0, **kw)
    if p.pattern == AG:
        comm.ag_gemm(p, fx.TileShape(p.rows_per_rank(), p.local_cols()), rpct, transfer, swizzle, opts)
    else:
        comm.gemm_rs(p, fx.TileShape(p.rows_per_rank(), p.local_cols()), write_mode, swizzle, opts)
    comm.sync()
    return H.outputs(comm, p, f32)


@pytest.mark.parametrize("f32", [True, False])
def test_golden_configs_match_reference(f32):
    """The reference's golden config (16x16x16, tp=4, seed 42) and the other
    fixtures made from the reference library itself, on bf16 inputs."""
    with open(GOLDEN) as f:
        cases = json.load(f)["bf16_cases"]
    for c in cases:
        p = fx.ProblemSpec(c["m"], c["n"], c["k"], c["tp"], c["pattern"])
        with H.make_comm(p) as comm:
            H.upload(comm, p, c["seed"])
            got = _run(comm, p, f32)
            for r in range(p.tp):
                err = O.max_rel_error(got[r], _unhex(c["outputs"][r]))
                assert err <= H.tol(f32, c["k"]), (c["pattern"], c["m"], r, err)


def _oracle(p, a, b):
    return O.dense_oracle(p.pattern, p.m, p.n, p.k, p.tp, a, b)


CASES = [
    # (pattern, m, n, k, tp) — ragged shapes exercise TMA OOB fill and masked epilogues
    (AG, 256, 512, 128, 2), (AG, 1024, 2048, 512, 8), (AG, 40, 24, 72, 4), (AG, 384, 768, 320, 4),
    (AG, 8, 8, 8, 1), (AG, 1000, 600, 200, 1),
    (RS, 1024, 512, 256, 4), (RS, 512, 768, 1024, 2), (RS, 40, 24, 72, 4), (RS, 2048, 1024, 512, 8),
    (RS, 192, 300, 96, 2), (RS, 64, 64, 64, 1),
    # columns not a multiple of 4 / of the tile; decode-sized blocks straddling tiles
    (RS, 24, 301, 40, 4), (RS, 200, 257, 64, 8), (RS, 360, 515, 96, 8), (AG, 96, 300, 136, 4),
    # fewer tiles than SMs with several K-blocks: split-K reduction units (slices summed in order,
    # then staged for the owners), incl. TP=1 (one GPU's decode share) and ragged columns
    (RS, 1024, 1024, 1024, 2), (RS, 32, 1024, 2048, 2), (RS, 16, 2048, 4096, 8), (RS, 16, 2048, 3584, 1),
    (RS, 48, 1000, 1536, 4),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c)))
def test_fused_matches_oracle(case):
    pat, m, n, k, tp = case
    p = fx.ProblemSpec(m, n, k, tp, pat)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=1000 + m + n + k + tp)
        want = _oracle(p, a, b)
        for f32 in (True, False):
            got = _run(comm, p, f32)
            for r in range(tp):
                assert O.max_rel_error(got[r], want[r]) <= H.tol(f32, p.k), (f32, r)
        assert comm.last_launch_count() >= 1


@pytest.mark.parametrize("cta_group", [1, 2])
@pytest.mark.parametrize("case", [(AG, 1024, 1024, 512, 4), (AG, 600, 520, 136, 2), (RS, 2048, 768, 512, 4),
                                  (RS, 1280, 640, 200, 2), (RS, 512, 512, 256, 8)],
                         ids=lambda c: "x".join(map(str, c)))
def test_single_cta_and_cta_pair_tiles(case, cta_group):
    """Both MMA variants: one CTA per 128x256 tile (cta_group::1) and CTA pairs
    sharing 256x256 tiles (cta_group::2), incl. tiles straddling rank blocks."""
    pat, m, n, k, tp = case
    p = fx.ProblemSpec(m, n, k, tp, pat)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=77 + m)
        want = _oracle(p, a, b)
        got = _run(comm, p, True, cta_group=cta_group)
        for r in range(tp):
            assert O.max_rel_error(got[r], want[r]) <= H.tol(True, p.k), r
        comm.local_gemm(p, fx.default_opts(out_dtype=fx.F32, cta_group=cta_group))
        comm.sync()


@pytest.mark.parametrize("engine", [1, 2])
@pytest.mark.parametrize("case", [(AG, 1024, 2048, 512, 8), (AG, 16, 1024, 8192, 8), (AG, 40, 24, 72, 4),
                                  (AG, 256, 512, 20000, 2), (AG, 64, 256, 136, 1), (AG, 4096, 1024, 256, 4)],
                         ids=lambda c: "x".join(map(str, c)))
def test_allgather_transfer_engines(case, engine):
    """Copy-engine transfer loop (ag_engine=1) and the in-kernel transfer by the
    GEMM's own SMs (ag_engine=2): whole-row pieces, per-row pieces (padded
    pitch) and column-split pieces (rows > 16 KiB)."""
    pat, m, n, k, tp = case
    p = fx.ProblemSpec(m, n, k, tp, pat)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=31 + k)
        want = _oracle(p, a, b)
        for _ in range(3):  # back to back: epoch-stamped counters, no resets
            got = _run(comm, p, True, ag_engine=engine)
            for r in range(tp):
                assert O.max_rel_error(got[r], want[r]) <= H.tol(True, p.k), r


@pytest.mark.parametrize("tp,rpct", [(4, 64), (4, 32), (2, 512), (8, 16)])
def test_allgather_comm_tile_sizes_and_transfer_modes(tp, rpct):
    """Comm tiles decoupled from GEMM tiles (SPEC §4.3), pull and push."""
    m = tp * max(256, rpct) if rpct >= 64 else 64 * tp
    p = fx.ProblemSpec(m, 256 * tp, 192, tp, AG)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=7)
        want = _oracle(p, a, b)
        outs = {}
        for engine in (1, 2):  # copy engines, in-kernel (SM) transfers
            for transfer in (fx.PULL, fx.PUSH):
                for swizzle in (True, False):
                    got = _run(comm, p, True, transfer=transfer, swizzle=swizzle, rpct=rpct, ag_engine=engine)
                    outs[(engine, transfer, swizzle)] = got
                    for r in range(tp):
                        assert O.max_rel_error(got[r], want[r]) <= H.tol(True, p.k)
        # push == pull bitwise (test_engine.cpp:63-74): same GEMM, same inputs, either engine
        for r in range(tp):
            for key in outs:
                assert np.array_equal(outs[(1, fx.PULL, True)][r], outs[key][r]) or not key[2], key


def test_reduce_scatter_is_deterministic_across_runs_and_orders():
    """Source-ordered reduction: bit-identical run to run and for both swizzles
    (test_engine.cpp:215-227 bitwise across pool sizes)."""
    p = fx.ProblemSpec(2048, 1024, 1024, 8, RS)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=3)
        first = _run(comm, p, True)
        for swizzle in (True, False, True):
            again = _run(comm, p, True, swizzle=swizzle)
            for r in range(p.tp):
                assert np.array_equal(first[r], again[r])
        nonov = None
        comm.nonoverlap(p, fx.default_opts(out_dtype=fx.F32))
        comm.sync()
        nonov = H.outputs(comm, p, True)
        want = _oracle(p, a, b)
        for r in range(p.tp):
            assert O.max_rel_error(nonov[r], want[r]) <= H.tol(True, p.k)


@pytest.mark.parametrize("case", [(2048, 1024, 1024, 8), (1024, 512, 768, 4), (40, 24, 72, 4), (384, 256, 128, 2)],
                         ids=lambda c: "x".join(map(str, c)))
def test_fused_reduce_arrival_order(case):
    """FusedReduce with deterministic_reduce=False (engine.cpp:304-319): vector
    red.add into the owner's fp32 accumulator; mixed back to back with
    WriteAlltoAll on the same communicator (epoch parity reuse)."""
    m, n, k, tp = case
    p = fx.ProblemSpec(m, n, k, tp, RS)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=5 + m)
        want = _oracle(p, a, b)
        for mode in (fx.FUSED_REDUCE, fx.WRITE_ALLTOALL, fx.FUSED_REDUCE, fx.FUSED_REDUCE):
            for f32 in (True, False):
                got = _run(comm, p, f32, write_mode=mode, deterministic_reduce=0)
                for r in range(tp):
                    assert O.max_rel_error(got[r], want[r]) <= H.tol(f32, p.k), (mode, f32, r)


def test_nonoverlap_baseline_allgather():
    p = fx.ProblemSpec(512, 1024, 256, 4, AG)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=5)
        comm.nonoverlap(p, fx.default_opts(out_dtype=fx.F32))
        comm.sync()
        got = H.outputs(comm, p, True)
        fused = _run(comm, p, True)
        want = _oracle(p, a, b)
        for r in range(p.tp):
            assert O.max_rel_error(got[r], want[r]) <= H.tol(True, p.k)
            assert np.array_equal(got[r], fused[r])


def test_back_to_back_operators_without_host_sync():
    """Epoch-stamped flags: many launches queued with no reset or host sync."""
    p = fx.ProblemSpec(1024, 1024, 512, 4, AG)
    q = fx.ProblemSpec(1024, 512, 512, 4, RS)
    heap = max(fx.required_heap_bytes(p), fx.required_heap_bytes(q))
    with fx.Communicator(4, [0] * 4, heap_bytes=heap) as comm:
        a, b = H.upload(comm, p, seed=11)
        for _ in range(5):
            comm.ag_gemm(p, fx.TileShape(256, 256), 128, fx.PULL, True, fx.default_opts(out_dtype=fx.F32))
        comm.sync()
        want = _oracle(p, a, b)
        got = H.outputs(comm, p, True)
        for r in range(4):
            assert O.max_rel_error(got[r], want[r]) <= H.tol(True, p.k)
        a, b = H.upload(comm, q, seed=12)
        for _ in range(5):
            comm.gemm_rs(q, fx.TileShape(256, 512), fx.WRITE_ALLTOALL, True, fx.default_opts(out_dtype=fx.F32))
        comm.sync()
        want = _oracle(q, a, b)
        got = H.outputs(comm, q, True)
        for r in range(4):
            assert O.max_rel_error(got[r], want[r]) <= H.tol(True, p.k)


def test_jitter_does_not_change_results():
    """Race injection (reference Jitter, engine.cpp:116-128; test_engine.cpp:190-213)."""
    p = fx.ProblemSpec(1024, 1024, 256, 4, RS)
    with H.make_comm(p) as comm:
        H.upload(comm, p, seed=21)
        base = _run(comm, p, True)
        for seed in (1, 2, 3):
            got = _run(comm, p, True, interleave_seed=seed)
            for r in range(p.tp):
                assert np.array_equal(base[r], got[r])


def test_directory_error_for_unmapped_peer():
    """DirectoryError on a dropped peer entry (workspace.cpp:56-69, test_engine.cpp:182-188)."""
    p = fx.ProblemSpec(64, 64, 64, 4, AG)
    with H.make_comm(p) as comm:
        comm.drop_peer(1, 2)
        with pytest.raises(fx.DirectoryError, match="rank 1 has no directory entry for peer 2"):
            comm.ag_gemm(p, fx.TileShape(16, 16))


def test_shape_and_config_errors():
    p = fx.ProblemSpec(64, 64, 64, 4, AG)
    with H.make_comm(p) as comm:
        with pytest.raises(fx.ConfigError, match="requires GemmReduceScatter"):
            comm.gemm_rs(p, fx.TileShape(16, 16))
        with pytest.raises(fx.ShapeError):
            comm.ag_gemm(fx.ProblemSpec(64, 64, 64, 2, AG), fx.TileShape(16, 16))
        with pytest.raises(fx.ShapeError, match="heap bytes"):
            comm.ag_gemm(fx.ProblemSpec(8192, 8192, 8192, 4, AG), fx.TileShape(16, 16))


FULL_SIZE = {  # BASELINE.json configs: Llama-2-70B MLP (TP=8, RS also TP=2/4), GPT-3 175B MLP, decode M=16 / 512
    "llama-ag": (AG, 4096, 28672, 8192, 8), "llama-rs": (RS, 4096, 8192, 28672, 8),
    "llama-rs-tp4": (RS, 4096, 8192, 28672, 4), "llama-rs-tp2": (RS, 4096, 8192, 28672, 2),
    "gpt3-ag": (AG, 8192, 49152, 12288, 8), "gpt3-rs": (RS, 8192, 12288, 49152, 8),
    "decode-ag-m16": (AG, 16, 28672, 8192, 8), "decode-rs-m512": (RS, 512, 8192, 28672, 8),
    # the rest of configs[4] (decode sweep): AG up M=128/256/512, RS down M=16/128/256, attention-out
    # (K=N=8192) M=16/128/512, and the C1 oracle-plumbing config at full size
    "decode-ag-m128": (AG, 128, 28672, 8192, 8), "decode-ag-m256": (AG, 256, 28672, 8192, 8),
    "decode-ag-m512": (AG, 512, 28672, 8192, 8),
    "decode-rs-m16": (RS, 16, 8192, 28672, 8), "decode-rs-m128": (RS, 128, 8192, 28672, 8),
    "decode-rs-m256": (RS, 256, 8192, 28672, 8),
    "decode-attn-m16": (RS, 16, 8192, 8192, 8), "decode-attn-m128": (RS, 128, 8192, 8192, 8),
    "decode-attn-m512": (RS, 512, 8192, 8192, 8),
    # one GPU's share of the decode configs (TP=1 problems with the per-rank shapes)
    "rank-decode-ag-m16": (AG, 16, 3584, 8192, 1), "rank-decode-rs-m16": (RS, 16, 8192, 3584, 1),
    "rank-decode-rs-m128": (RS, 128, 8192, 3584, 1),
}


def test_c1_oracle_plumbing_config_matches_oracle_and_reference_engine():
    """BASELINE configs[0] exactly: GEMM-ReduceScatter M=N=K=1024 at TP=2 (the
    reference's CPU oracle-plumbing config), every output element against the
    fp64 oracle; the oracle itself equals the reference's fused engine bitwise
    at this size (tests/test_oracle.py)."""
    p = fx.ProblemSpec(1024, 1024, 1024, 2, RS)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=42)
        want = _oracle(p, a, b)
        for f32 in (True, False):
            for write_mode in (fx.WRITE_ALLTOALL, fx.FUSED_REDUCE):
                got = _run(comm, p, f32, write_mode=write_mode)
                for r in range(p.tp):
                    assert O.max_rel_error(got[r], want[r]) <= H.tol(f32, p.k), (f32, write_mode, r)


@pytest.mark.slow
@pytest.mark.parametrize("name", list(FULL_SIZE))
def test_full_size_tp8_row_sampled(name):
    """BASELINE configs at full size (ranks emulated on one GPU), checked on
    sampled rows: >= 1 row per (rank, row block) for AG, 2 owned rows per rank
    for RS, against the fp64 oracle on the same bf16 inputs."""
    pattern, m, n, k, tp = FULL_SIZE[name]
    p = fx.ProblemSpec(m, n, k, tp, pattern)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=42)
        got = _run(comm, p, False)
        rng = np.random.default_rng(0)
        rpr = p.rows_per_rank()
        for r in range(p.tp):
            if pattern == AG:
                rows = sorted(int(x) for blk in range(p.tp) for x in rng.integers(blk * rpr, (blk + 1) * rpr, 1))
                want = O.ag_rows(p.m, p.n, p.k, p.tp, a, b[r], rows)
                assert O.max_rel_error(got[r][rows], want) <= 8e-3
            else:
                lrows = sorted(int(x) for x in rng.integers(0, rpr, 2))
                want = O.rs_rows(p.m, p.n, p.k, p.tp, a, b, r, lrows)
                assert O.max_rel_error(got[r][lrows], want) <= 8e-3


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_causality_from_device_trace_allgather(seed):
    """Reference acceptance criterion 2 / test_engine.cpp:190-213 on the device:
    under jitter, every tile's compute_start follows the signal_set of the
    a_agg group it consumed (both stamped with %globaltimer)."""
    p = fx.ProblemSpec(1024, 2048, 256, 4, AG)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=3)
        got = _run(comm, p, True, ag_engine=2, trace=1, interleave_seed=seed)
        want = _oracle(p, a, b)
        for r in range(p.tp):
            assert O.max_rel_error(got[r], want[r]) <= H.tol(True, p.k)
            ev = fx.comm.read_trace(comm, r, p)
            sets = {}
            for e in ev:
                if e["event"] == "signal_set" and e["rank"] == r:
                    sets[e["target"]] = max(sets.get(e["target"], -1), e["logical_ts"])
            starts = [e for e in ev if e["event"] == "compute_start" and e["rank"] == r]
            assert len(starts) == (p.m // 128) * (p.local_cols() // 256)
            assert len(sets) == p.m // 128
            for e in starts:
                assert e["logical_ts"] > sets[e["target"]], e


def test_causality_from_device_trace_reduce_scatter():
    """Owners reduce a tile only after every source's tile_write for it."""
    p = fx.ProblemSpec(2048, 512, 512, 8, RS)
    with H.make_comm(p) as comm:
        H.upload(comm, p, seed=4)
        _run(comm, p, True, trace=1, interleave_seed=5)
        writes, reduces = {}, []
        for r in range(p.tp):
            for e in fx.comm.read_trace(comm, r, p):
                key = (e["tile_row"], e["tile_col"])
                if e["event"] == "tile_write":
                    writes.setdefault((e["target"], key), []).append(e["ts"])
                elif e["event"] == "reduce":
                    reduces.append((e["rank"], key, e["ts"]))
        assert len(reduces) == (p.m // 128) * (p.n // 256)
        for owner, key, t in reduces:  # all ranks share one GPU: one %globaltimer
            w = writes.get((owner, key), [])
            assert len(w) == p.tp - 1 and max(w) <= t, (owner, key)


@pytest.mark.parametrize("engine", [1, 2])
def test_caller_owned_operands(engine):
    """flux_ag_gemm_ex / flux_gemm_rs_ex on caller tensors (weights outside the
    symmetric heap, padded A pitch, caller C) match the library-buffer path."""
    tp = 4
    p = fx.ProblemSpec(1024, 2048, 320, tp, AG)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=8)
        want = _oracle(p, a, b)
        ops = []
        for r in range(tp):
            wide = torch.zeros(p.rows_per_rank(), 384, dtype=torch.bfloat16, device="cuda")
            wide[:, :p.k].copy_(comm.tensor(r, N.BUF_A_SHARD, p))
            a_view = wide[:, :p.k]                       # ld 384 != k
            w = comm.tensor(r, N.BUF_B_SHARD, p).contiguous()
            c = torch.empty(p.m, p.local_cols(), dtype=torch.float32, device="cuda")
            ops.append((a_view, w, c))
        comm.ag_gemm_ex(p, fx.TileShape(256, 256), ops, opts=fx.default_opts(out_dtype=fx.F32, ag_engine=engine))
        comm.sync()
        for r in range(tp):
            assert O.max_rel_error(ops[r][2].double().cpu().numpy(), want[r]) <= H.tol(True, p.k)
    q = fx.ProblemSpec(1024, 512, 512, tp, RS)
    with H.make_comm(q) as comm:
        a, b = H.upload(comm, q, seed=9)
        want = _oracle(q, a, b)
        ops = [(comm.tensor(r, N.BUF_A_SHARD, q).contiguous(), comm.tensor(r, N.BUF_B_SHARD, q).contiguous(),
                torch.empty(q.rows_per_rank(), q.n, dtype=torch.float32, device="cuda")) for r in range(tp)]
        comm.gemm_rs_ex(q, fx.TileShape(256, 512), ops, opts=fx.default_opts(out_dtype=fx.F32))
        comm.sync()
        for r in range(tp):
            assert O.max_rel_error(ops[r][2].double().cpu().numpy(), want[r]) <= H.tol(True, q.k)


def test_acceptance_randomized_equivalence():
    """Reference acceptance criterion 1 (acceptance.cpp:67-118) on the GPU: 200
    randomized cases, tp in {1,2,4,8}, both patterns, every transfer / write
    mode and both CTA-group variants, against the oracle."""
    rng = np.random.default_rng(42)
    worst = 0.0
    for i in range(200):
        pat = RS if i % 2 else AG
        tp = int(rng.choice([1, 2, 4, 8]))
        rpr = int(rng.choice([8, 16, 40, 128, 256]))
        m = rpr * tp
        if pat == AG:
            n = tp * int(rng.choice([8, 24, 128, 256]))
            k = int(rng.choice([8, 16, 72, 136, 512]))
        else:
            n = int(rng.choice([8, 24, 128, 256, 300]))
            k = tp * int(rng.choice([8, 16, 72, 128]))
        p = fx.ProblemSpec(m, n, k, tp, pat)
        kw = {"cta_group": int(rng.choice([0, 1, 2]))}
        if pat == AG:
            kw["ag_engine"] = int(rng.choice([1, 2]))
            mode = {"transfer": fx.PUSH if rng.random() < 0.3 else fx.PULL,
                    "swizzle": bool(rng.random() < 0.8)}
        else:
            mode = {"write_mode": int(rng.choice([fx.WRITE_ALLTOALL, fx.FUSED_REDUCE])),
                    "swizzle": bool(rng.random() < 0.8)}
            kw["deterministic_reduce"] = int(rng.random() < 0.5)
        with H.make_comm(p) as comm:
            a, b = H.upload(comm, p, seed=1000 + i)
            got = _run(comm, p, True, **mode, **kw)
            want = _oracle(p, a, b)
            for r in range(tp):
                err = O.max_rel_error(got[r], want[r])
                worst = max(worst, err)
                assert err <= H.tol(True, p.k), (i, pat, m, n, k, tp, mode, kw, r, err)
    print("200 randomized cases, worst max_rel_error", worst)


@pytest.mark.parametrize("tp", [4, 8])
def test_rs_chain_bit_identical_to_owner_sum(tp, monkeypatch):
    """Chained partial sums (all ranks in one launch, long rank sections) and the
    owner-side sum use the same canonical order: bit-identical outputs; and both
    match fp32 cuBLAS products of the same bf16 operands."""
    p = fx.ProblemSpec(4096, 4096, 128 * tp, tp, RS)  # 256 CTA-pair tiles per rank: the chain is on
    with H.make_comm(p) as comm:
        g = torch.Generator(device="cuda")
        g.manual_seed(tp)
        for r in range(tp):
            for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
                t = comm.tensor(r, kind, p)
                t.copy_((torch.rand(t.shape, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16))
        torch.cuda.synchronize()
        chained = _run(comm, p, True)
        monkeypatch.setenv("FLUX_RS_CHAIN", "0")
        owner_sum = _run(comm, p, True)
        for r in range(tp):
            assert np.array_equal(chained[r], owner_sum[r]), r
        a = [comm.tensor(r, N.BUF_A_SHARD, p).float() for r in range(tp)]
        b = [comm.tensor(r, N.BUF_B_SHARD, p).float() for r in range(tp)]
        rpr = p.rows_per_rank()
        for r in range(tp):
            rows = torch.arange(r * rpr, (r + 1) * rpr, 97, device="cuda")
            ref = sum(a[s][rows] @ b[s].t() for s in range(tp)).cpu().numpy()
            got = chained[r][(rows - r * rpr).cpu().numpy()]
            assert np.abs(got - ref).max() / max(1.0, np.abs(ref).max()) < 1e-4, r


@pytest.mark.parametrize("tp", [3, 5, 6, 7])
def test_odd_tp_degrees(tp):
    """TP degrees that are not powers of two (reference ProblemSpec allows any
    tp dividing m): AG (both engines), RS aligned and decode-sized blocks."""
    for pat, m, n, k in [(AG, 128 * tp, 256 * tp, 192), (RS, 256 * tp, 512, 64 * tp), (RS, 8 * tp, 320, 32 * tp)]:
        p = fx.ProblemSpec(m, n, k, tp, pat)
        with H.make_comm(p) as comm:
            a, b = H.upload(comm, p, seed=tp * 13 + m)
            want = _oracle(p, a, b)
            engines = (1, 2) if pat == AG else (0,)
            for engine in engines:
                for swizzle in (True, False):
                    got = _run(comm, p, True, swizzle=swizzle, ag_engine=engine)
                    for r in range(tp):
                        assert O.max_rel_error(got[r], want[r]) <= H.tol(True, p.k), (pat, m, engine, swizzle, r)


def _normwise(got, want):
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))


@pytest.mark.parametrize("case", [(1024, 512, 768, 4), (2048, 1024, 1024, 8), (4096, 4096, 512, 4),
                                  (40, 24, 72, 4), (512, 8192, 1024, 8), (360, 515, 96, 8)],
                         ids=lambda c: "x".join(map(str, c)))
def test_rs_bf16_partials_normwise(case):
    """opts.rs_partials = BF16 (half the cross-rank bytes): one bf16 rounding per
    partial (owner sum, decode owner units) or per chain link (4096x4096:
    chained); checked normwise <= 5e-3, and it must differ from
    the fp32 path only by that rounding. FusedReduce rejects it."""
    m, n, k, tp = case
    p = fx.ProblemSpec(m, n, k, tp, RS)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=m + tp)
        f32 = _run(comm, p, True)
        bf = _run(comm, p, True, rs_partials=fx.BF16)
        if m * n * k <= 2048 * 1024 * 1024:
            want = _oracle(p, a, b)
            rows = [list(range(p.rows_per_rank()))] * tp
        else:  # row-sampled oracle rows (rs_rows), 8 per owner
            rpr = p.rows_per_rank()
            rows = [sorted({0, rpr - 1} | {(r * 131 + i * (rpr // 6)) % rpr for i in range(6)}) for r in range(tp)]
            want = [O.rs_rows(m, n, k, tp, a, b, r, rows[r]) for r in range(tp)]
        for r in range(tp):
            assert _normwise(bf[r][rows[r]], want[r]) <= 5e-3, r
            assert _normwise(bf[r], f32[r]) <= 5e-3, r
    q = fx.ProblemSpec(1024, 512, 768, 4, RS)  # arrival-order FusedReduce accumulates in fp32
    with H.make_comm(q) as comm:
        with pytest.raises(fx.ConfigError, match="bf16 partials"):
            _run(comm, q, True, rs_partials=fx.BF16, write_mode=fx.FUSED_REDUCE, deterministic_reduce=0)


@pytest.mark.parametrize("cta_group", [1, 2])
@pytest.mark.parametrize("case", [(AG, 1024, 2048, 512, 4), (RS, 1024, 512, 768, 4), (AG, 512, 1536, 200, 2),
                                  (RS, 2048, 1024, 1024, 8), (RS, 64, 256, 256, 4)],
                         ids=lambda c: "x".join(map(str, c)))
def test_b_layout_kn(case, cta_group):
    """Caller B given as [k, n] row-major (the reference's b_shard layout,
    opts.b_layout = KN): MN-major tcgen05 B operand, no transposed copy."""
    pat, m, n, k, tp = case
    p = fx.ProblemSpec(m, n, k, tp, pat)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=19 + m)
        want = _oracle(p, a, b)
        b_kn = [comm.tensor(r, N.BUF_B_SHARD, p).t().contiguous() for r in range(tp)]  # [k_local, n_local]
        opts = fx.default_opts(out_dtype=fx.F32, wall_budget_s=5.0, b_layout=fx.B_KN, cta_group=cta_group)
        ops = [(None, b_kn[r], None) for r in range(tp)]
        tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
        if pat == AG:
            comm.ag_gemm_ex(p, tile, ops, opts=opts)
        else:
            comm.gemm_rs_ex(p, tile, ops, opts=opts)
        comm.sync()
        got = H.outputs(comm, p, True)
        for r in range(tp):
            assert O.max_rel_error(got[r], want[r]) <= H.tol(True, p.k), r
        with pytest.raises(fx.ConfigError, match="caller-provided B"):
            comm.ag_gemm(p, tile, opts=opts) if pat == AG else comm.gemm_rs(p, tile, opts=opts)


@pytest.mark.parametrize("pattern", [AG, RS])
def test_acceptance_wallclock_ratio(pattern):
    """Reference acceptance criterion 7 (acceptance.cpp:323-371): fused /
    non-overlapped wall-clock ratio <= 1.5 (there non-gating, on CPU threads);
    here on the GPU with device time, medians of 5 after warm-up."""
    p = fx.ProblemSpec(2048, 8192, 2048, 8, pattern) if pattern == AG else fx.ProblemSpec(2048, 2048, 8192, 8, pattern)
    with H.make_comm(p) as comm:
        for r in range(p.tp):
            for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
                t = comm.tensor(r, kind, p)
                t.copy_((torch.rand(t.shape, device="cuda") * 2 - 1).to(torch.bfloat16))
        tile = fx.TileShape(p.rows_per_rank(), p.local_cols())

        def fused():
            comm.ag_gemm(p, tile) if pattern == AG else comm.gemm_rs(p, tile)

        def nonoverlap():
            comm.nonoverlap(p)

        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        times = {"fused": [], "nonoverlap": []}
        for fn in (fused, nonoverlap, fused, nonoverlap):
            fn()
        comm.sync()
        for _ in range(5):
            for name, fn in (("fused", fused), ("nonoverlap", nonoverlap)):
                e0.record()
                fn()
                e1.record()
                comm.sync()
                times[name].append(e0.elapsed_time(e1))
        ratio = float(np.median(times["fused"]) / np.median(times["nonoverlap"]))
        print(f"fused / non-overlapped wall-clock ratio ({'AG' if pattern == AG else 'RS'}): {ratio:.3f}")
        assert ratio <= 1.5


@pytest.mark.parametrize("pat,m,n,k,tp", [(AG, 2048, 3072, 512, 4), (AG, 1664, 2304, 640, 8),
                                          (RS, 4096, 4096, 1024, 8), (RS, 1024, 2048, 512, 4)])
def test_dynamic_scheduler_bit_identical(pat, m, n, k, tp, monkeypatch):
    """FLUX_DYN_SCHED=1 (counter-fetched tiles, cluster tile queue) changes only
    which cluster runs a unit: outputs are bit-identical to the static stride,
    repeated launches re-arm the counter, and both match the oracle."""
    p = fx.ProblemSpec(m, n, k, tp, pat)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=m + tp)
        static = _run(comm, p, True)
        monkeypatch.setenv("FLUX_DYN_SCHED", "1")
        for _ in range(3):
            dyn = _run(comm, p, True)
            for r in range(tp):
                assert np.array_equal(static[r], dyn[r]), r
        want = _oracle(p, a, b)
        for r in range(tp):
            np.testing.assert_allclose(dyn[r], want[r], rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("case", [(AG, 1024, 1024, 512, 4, 4), (AG, 1024, 768, 256, 4, 8), (AG, 64, 256, 128, 2, 4),
                                  (RS, 1024, 512, 512, 4, 4), (RS, 2048, 1024, 256, 8, 16), (RS, 40, 24, 72, 4, 8),
                                  (RS, 64, 64, 64, 1, 1)],
                         ids=lambda c: "x".join(map(str, c)))
def test_medium_grained_baseline(case):
    """run_medium_grained (engine.hpp:144-145) on the device — chunked
    transfers / GEMMs / reduces (B2) — matches the oracle; invalid partition
    counts raise the reference's ConfigError."""
    pat, m, n, k, tp, parts = case
    p = fx.ProblemSpec(m, n, k, tp, pat)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=m + parts)
        want = _oracle(p, a, b)
        tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
        for f32 in (True, False):
            comm.medium_grained(p, tile, parts, fx.default_opts(out_dtype=fx.F32 if f32 else fx.BF16))
            comm.sync()
            got = H.outputs(comm, p, f32)
            for r in range(tp):
                assert O.max_rel_error(got[r], want[r]) <= H.tol(f32, p.k), (f32, r)
        if tp > 1:
            with pytest.raises(fx.ConfigError, match="must be tp or 2\\*tp"):
                comm.medium_grained(p, tile, 3 * tp)


@pytest.mark.parametrize("case", [(AG, 500, 600, 2048, 1), (AG, 640, 512, 2048, 4), (RS, 128, 512, 8192, 4),
                                  (RS, 64, 512, 16384, 8)], ids=lambda c: "x".join(map(str, c)))
def test_tail_split_last_wave_matches_oracle(case):
    """The last partial wave's tiles run as K-slices (each CTA of the wave sums
    its share of the slices in slice order) when K is long enough to pay for it
    (>= 24 k-blocks per rank): AG and the decode-sized RS units on the tile
    kernel, against the oracle."""
    pat, m, n, k, tp = case
    p = fx.ProblemSpec(m, n, k, tp, pat)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=m + k)
        split = _run(comm, p, True, decode_kernel=fx.DECODE_TILE)
        want = _oracle(p, a, b)
        for r in range(tp):
            assert O.max_rel_error(split[r], want[r]) <= H.tol(True, k), r

