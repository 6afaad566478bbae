"""bench.py's roofline arithmetic: the bound of each
BASELINE config is the slowest of tensor-core, HBM and NVLink time at peak."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

PK = {"bf16_tflops": 1665.3, "hbm_gbs": 6554.0}


def _bound(pattern, m, n, k, tp, emulated):
    r = bench.roofline_of(bench.roofline_work(pattern, m, n, k, tp, emulated), 1.0, PK, "test")
    return r


@pytest.mark.parametrize("wl,bound,us", [
    ((0, 4096, 28672, 8192, 8), "tensor", 144.4),   # L-AG TP=8, one rank
    ((1, 4096, 8192, 28672, 8), "tensor", 144.4),   # L-RS TP=8
    ((1, 4096, 8192, 28672, 2), "tensor", 577.7),   # L-RS TP=2
    ((0, 8192, 49152, 12288, 8), "tensor", 742.8),  # G-AG
    ((1, 1024, 1024, 1024, 2), "nvlink", 2.33),     # C1 (fp32 partials)
    ((1, 512, 8192, 8192, 8), "nvlink", 16.31),     # decode attn-out M=512
])
def test_survey_table_per_rank(wl, bound, us):
    r = _bound(*wl, emulated=False)
    assert r["bound"] == bound
    assert abs(r["roofline_us"] - us) / us < 0.01, r["terms_us"]


def test_decode_is_hbm_bound():
    # D AG up / RS down, M=16 at TP=8: the 58.7 MB weight shard dominates (~9 us)
    for wl in ((0, 16, 28672, 8192, 8), (1, 16, 8192, 28672, 8)):
        r = _bound(*wl, emulated=False)
        assert r["bound"] == "hbm" and 8.9 < r["roofline_us"] < 9.3, r["terms_us"]
    # one rank's share as a TP=1 problem (bench workloads rank-decode-*)
    r = _bound(1, 16, 8192, 3584, 1, emulated=True)
    assert r["bound"] == "hbm" and 8.9 < r["roofline_us"] < 9.3


def test_emulated_launch_counts_every_rank_and_no_nvlink():
    per_rank = bench.roofline_work(0, 4096, 28672, 8192, 8, emulated=False)
    launch = bench.roofline_work(0, 4096, 28672, 8192, 8, emulated=True)
    assert launch[0] == 8 * per_rank[0] and launch[1] == 8 * per_rank[1] and launch[2] == 0.0


def test_frac_is_roofline_time_over_kernel_time():
    work = bench.roofline_work(1, 16, 8192, 3584, 1, emulated=True)
    r = bench.roofline_of(work, 0.020, PK, "test")
    assert abs(r["frac"] - r["roofline_us"] / 20.0) < 1e-9
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
