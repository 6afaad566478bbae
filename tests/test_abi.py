"""The C-ABI library loads and exports every symbol include/flux_b200.h declares
(no compute calls: this runs without a GPU)."""
import os
import re
import subprocess

from paper_2406_06858_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flux_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(flux_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert "flux_ag_gemm" in syms and "flux_gemm_rs" in syms and "flux_comm_create_ipc" in syms
    assert len(syms) >= 25


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(flux_[a-z0-9_]+)$", out, flags=re.M))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    for s in declared_symbols():
        getattr(lib, s)


def test_python_binding_covers_the_header():
    assert sorted(N.EXPORTED) == declared_symbols()


def test_library_is_sm100a_and_uses_tcgen05():
    out = subprocess.run(["cuobjdump", "-sass", N.LIB_PATH], capture_output=True, text=True, check=True).stdout
    assert "UTCHMMA" in out  # tcgen05.mma
    assert "UTMALDG" in out  # TMA loads
    assert "LDTM" in out     # tcgen05.ld (TMEM -> registers)
    assert "LDGMC" in out    # multimem.ld_reduce (NVLS owner-side reduction in the switch)
    elf = subprocess.run(["cuobjdump", "-lelf", N.LIB_PATH], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in elf


def test_abi_version_and_defaults():
    lib = N.lib()
    assert lib.flux_abi_version() == N.ABI_VERSION == 8
    o = N.default_opts()
    assert o.activation == N.ACT_NONE and o.activation_grad == N.ACT_NONE and o.rs_partials == N.F32 and o.b_layout == N.B_NK
    assert o.graph_safe == 0
    assert o.deterministic_reduce == 1 and o.shift_offset == 1 and o.wall_budget_s == 10.0
    assert o.poll_budget == 10_000_000  # EngineOptions defaults (engine.hpp:65-72)


def test_nvls_host_contract():
    """NVLS options without a GPU: off by default, region size per problem,
    the probe answers with a reason, unknown option names are rejected."""
    import ctypes as C

    import pytest

    import paper_2406_06858_b200 as fx

    assert N.default_opts().nvls == N.NVLS_OFF
    assert C.sizeof(N.CommOpts) == 2 * C.sizeof(C.c_size_t)
    ag = fx.ProblemSpec(4096, 28672, 8192, 8, fx.ALLGATHER_GEMM)
    rs = fx.ProblemSpec(4096, 8192, 28672, 8, fx.GEMM_REDUCESCATTER)
    assert fx.nvls_required_bytes(ag) == 64 * 1024 + 4096 * 8192 * 2  # flags, then a_agg [m, k] bf16
    assert fx.nvls_required_bytes(rs) == 64 * 1024 + 2 * 4096 * 8192 * 4  # flags, then 2 parities of [m, n] fp32
    assert fx.nvls_required_bytes(fx.ProblemSpec(10, 16, 16, 4, fx.ALLGATHER_GEMM)) == 0  # invalid (m % tp)
    ok, why = fx.nvls_probe([0])
    assert isinstance(ok, bool) and why
    with pytest.raises(TypeError):
        fx.default_opts(nvls_mode=1)
