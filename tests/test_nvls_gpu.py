"""NVLS (NVLink SHARP multicast through the NVSwitch, flux_opts.nvls).

AllGather-GEMM: each rank pushes its own comm tiles once into every rank's
a_agg with multicast stores and stamps the tile's flag on every rank; the GEMM
tiles wait on the flags (Alg. 2). GEMM-RS: each source keeps its partial in its
own region and each owner reads the sum over all sources with
multimem.ld_reduce (the owners' reduction units, or the streaming decode
kernel's epilogue).

FLUX_NVLS_EMULATED runs the same protocol — layouts, flags, epochs, the
owner-side reduction — with unicast loops over the ranks' regions, so it is
checked against the CPU oracle with every rank on one GPU. FLUX_NVLS_MULTICAST
needs a multicast object over >= 2 GPUs (flux_nvls_probe); those tests skip
where the host does not expose one (a one-GPU box: cuMulticastCreate fails)."""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_2406_06858_b200 as fx  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import gpu_harness as H  # noqa: E402

AG, RS = fx.ALLGATHER_GEMM, fx.GEMM_REDUCESCATTER
EMU, MC = fx.NVLS_EMULATED, fx.NVLS_MULTICAST


def _run(comm, p, f32=True, rpct=0, **kw):
    kw.setdefault("wall_budget_s", 5.0)
    opts = fx.default_opts(out_dtype=fx.F32 if f32 else fx.BF16, **kw)
    tile = fx.TileShape(p.rows_per_rank(), p.local_cols())
    if p.pattern == AG:
        comm.ag_gemm(p, tile, rpct or p.rows_per_rank(), fx.PULL, True, opts)
    else:
        comm.gemm_rs(p, tile, fx.WRITE_ALLTOALL, True, opts)
    comm.sync()
    return H.outputs(comm, p, f32)


# (pattern, m, n, k, tp, rpct): tile kernel (M >= 256) and streaming decode
# kernel (M <= 64, one rank per launch is not required in emulation), ragged
# n / k, several comm tiles per rank block.
CASES = [(AG, 512, 1024, 512, 4, 64), (AG, 1024, 2048, 1024, 8, 0), (AG, 256, 600, 200, 2, 32),
         (AG, 16, 1024, 512, 8, 0), (AG, 64, 3584, 1024, 4, 8),
         (RS, 512, 1024, 512, 4, 0), (RS, 1024, 1024, 2048, 8, 0), (RS, 256, 520, 256, 2, 0),
         (RS, 16, 1024, 1024, 8, 0), (RS, 64, 2048, 512, 4, 0)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c)))
def test_nvls_emulated_matches_oracle(case):
    pat, m, n, k, tp, rpct = case
    p = fx.ProblemSpec(m, n, k, tp, pat)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=5)
        want = O.dense_oracle(pat, m, n, k, tp, a, b)
        for f32 in (True, False):
            got = _run(comm, p, f32, rpct, nvls=EMU)
            for r in range(tp):
                assert O.max_rel_error(got[r], want[r]) <= H.tol(f32, k), (f32, r)


def test_nvls_emulated_interleaves_with_regular_operators():
    """NVLS and regular operators alternate on one communicator (epoch-stamped
    flags, staging parities): every result stays right."""
    for pat, (m, n, k) in ((AG, (512, 1024, 256)), (RS, (512, 768, 512))):
        p = fx.ProblemSpec(m, n, k, 4, pat)
        with H.make_comm(p) as comm:
            a, b = H.upload(comm, p, seed=9)
            want = O.dense_oracle(pat, m, n, k, 4, a, b)
            for nv in (EMU, fx.NVLS_OFF, EMU, EMU, fx.NVLS_OFF):
                got = _run(comm, p, True, 64, nvls=nv)
                for r in range(4):
                    assert O.max_rel_error(got[r], want[r]) <= H.tol(True, k), (nv, r)


def test_nvls_emulated_bit_identical_under_jitter():
    """The emulated owner sum runs in rank order: results do not depend on
    tile timing (device jitter)."""
    p = fx.ProblemSpec(512, 1024, 512, 4, RS)
    with H.make_comm(p) as comm:
        H.upload(comm, p, seed=2)
        ref = _run(comm, p, True, nvls=EMU)
        for seed in (1, 7):
            got = _run(comm, p, True, nvls=EMU, interleave_seed=seed)
            for r in range(4):
                assert (got[r] == ref[r]).all(), (seed, r)


def test_nvls_dropped_flag_raises_deadlock_error():
    """A dropped multicast flag stamp leaves the tiles of that comm tile
    waiting: DeadlockError naming the signal; the next operator is right."""
    p = fx.ProblemSpec(512, 1024, 256, 4, AG)
    with H.make_comm(p) as comm:
        a, b = H.upload(comm, p, seed=4)
        comm.inject_fault(fx.FAULT_DROP_SIGNAL, 1, 3)  # rank 1's comm tile 3 (rows 192..255, rpct 64)
        with pytest.raises(fx.DeadlockError) as ei:
            _run(comm, p, True, 64, nvls=EMU, wall_budget_s=0.5)
        assert "waiting for signal 3" in str(ei.value), str(ei.value)
        got = _run(comm, p, True, 64, nvls=EMU)
        want = O.dense_oracle(AG, p.m, p.n, p.k, 4, a, b)
        for r in range(4):
            assert O.max_rel_error(got[r], want[r]) <= H.tol(True, p.k), r


def test_nvls_config_errors():
    p = fx.ProblemSpec(512, 1024, 256, 4, RS)
    with H.make_comm(p) as comm:
        H.upload(comm, p, seed=1)
        assert not comm.nvls
        with pytest.raises(fx.ConfigError, match="nvls_bytes"):
            _run(comm, p, True, nvls=MC)
        with pytest.raises(fx.ConfigError, match="WriteAlltoAll"):
            comm.gemm_rs(p, fx.TileShape(128, 1024), fx.FUSED_REDUCE, True,
                         fx.default_opts(nvls=EMU, deterministic_reduce=0))
        with pytest.raises(fx.ConfigError, match="fp32 partials"):
            _run(comm, p, True, nvls=EMU, rs_partials=fx.BF16)
        with pytest.raises(fx.ConfigError, match="graph_safe"):
            _run(comm, p, True, nvls=EMU, graph_safe=1)
    with pytest.raises(TypeError):
        fx.default_opts(nvls_mode=1)


def test_nvls_probe_reports_a_reason():
    ok, why = fx.nvls_probe([0])
    assert isinstance(ok, bool) and why
    if not ok:
        # The single-GPU comm cannot own a region either (needs tp >= 2, distinct GPUs).
        p = fx.ProblemSpec(256, 256, 128, 2, AG)
        with pytest.raises((fx.CudaError, fx.ConfigError)):
            fx.Communicator(2, [0, 0], heap_bytes=fx.required_heap_bytes(p) + (8 << 20),
                            nvls_bytes=fx.nvls_required_bytes(p))


def _multicast_devices(n):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs (have {torch.cuda.device_count()})")
    ok, why = fx.nvls_probe(list(range(n)))
    if not ok:
        pytest.skip(f"NVLS multicast not exposed on this host: {why}")
    return list(range(n))


@pytest.mark.parametrize("case", [(AG, 1024, 2048, 1024, 0), (RS, 1024, 1024, 2048, 0), (AG, 16, 1024, 512, 0),
                                  (RS, 16, 1024, 1024, 0)], ids=lambda c: "x".join(map(str, c)))
@pytest.mark.parametrize("tp", [2, 4, 8])
def test_nvls_multicast_matches_oracle(case, tp):
    devs = _multicast_devices(tp)
    pat, m, n, k, rpct = case
    p = fx.ProblemSpec(m, n, k, tp, pat)
    comm = fx.Communicator(tp, devs, heap_bytes=max(fx.required_heap_bytes(p), 8 << 20),
                           nvls_bytes=fx.nvls_required_bytes(p))
    with comm:
        assert comm.nvls
        a, b = H.upload(comm, p, seed=6)
        want = O.dense_oracle(pat, m, n, k, tp, a, b)
        for _ in range(3):
            got = _run(comm, p, True, rpct, nvls=MC)
            for r in range(tp):
                assert O.max_rel_error(got[r], want[r]) <= H.tol(True, k), r
