"""Simulator-machine calibration arithmetic (paper_2406_06858_b200.calibrate):
the fits recover known parameters from synthetic measurements generated with
the reference's own model equations (sim.cpp:47-83), and the written machine
obeys MachineModel::validate (sim.cpp:52-57)."""
import pytest

from paper_2406_06858_b200 import calibrate as CAL
from paper_2406_06858_b200._native import ConfigError


def test_compute_fit_recovers_wave_model():
    truth = CAL.MachineModel(sm_count=148, flops_per_us=7.5e6, launch_overhead_us=6.0)
    tm, tn, k = 128, 256, 8192
    samples = [(tiles, truth.gemm_nonsplit_us(tiles, tm, tn, k)) for tiles in (148, 296, 444, 592, 1000)]
    launch, rate = CAL.fit_compute(samples, 148, tm, tn, k)
    assert launch == pytest.approx(6.0, rel=1e-9)
    assert rate == pytest.approx(7.5e6, rel=1e-9)


def test_link_fit():
    samples = [(b, 3.0 + b / 2.5e6) for b in (1 << 20, 4 << 20, 16 << 20, 64 << 20)]
    lat, bw = CAL.fit_link(samples)
    assert lat == pytest.approx(3.0, rel=1e-9)
    assert bw == pytest.approx(2.5e6, rel=1e-9)


def test_split_efficiency_fit():
    se = CAL.SplitEfficiency(exponent=0.2, floor=0.3)
    t_full = 1000.0
    chunks = {p: (t_full / p) / se(1.0 / p) for p in (2, 4, 8)}
    fit = CAL.fit_split_efficiency(CAL.split_efficiency_samples(t_full, chunks))
    assert fit.exponent == pytest.approx(0.2, rel=1e-9)
    assert fit(1.0) == 1.0
    for p in (2, 4, 8):
        assert fit(1.0 / p) == pytest.approx(se(1.0 / p), rel=1e-9)


def test_validate_and_schema():
    m = CAL.MachineModel(sm_count=148, flops_per_us=7e6, launch_overhead_us=5.0, link_bw_bytes_per_us=9e5,
                         link_latency_us=2.0, bytes_per_element=2)
    cfg = CAL.reference_config(m, {"m": 4096, "n": 28672, "k": 8192, "tp": 8, "pattern": "AllGatherGemm"},
                               {"tm": 128, "tn": 256}, {"gpu": "test"})
    mj = cfg["config"]["machine"]
    assert set(mj) == {"sm_count", "flops_per_us", "launch_overhead_us", "link_bw_bytes_per_us", "link_latency_us",
                       "inter_node_bw_bytes_per_us", "bytes_per_element", "topology", "split_efficiency"}
    assert set(mj["split_efficiency"]) == {"exponent", "floor"}
    with pytest.raises(ConfigError):
        CAL.MachineModel(sm_count=0).validate()
    with pytest.raises(ConfigError):
        CAL.MachineModel(link_latency_us=-1.0).validate()
    with pytest.raises(ValueError):
        CAL.fit_compute([(148, 10.0), (296, 5.0)], 148, 128, 256, 64)
