"""Fit the reference simulator's MachineModel from measurements on this GPU.

The reference's analytic simulator (`core/include/overlap/sim.hpp:19-42`,
`core/src/sim.cpp:47-83,457-475`) models a rank as `sm_count` tile slots, each
computing a (tm x tn) tile in `2*tm*tn*local_k / flops_per_us` microseconds,
plus a per-kernel `launch_overhead_us`, a link of `link_bw_bytes_per_us` with
`link_latency_us` per transfer, and a `SplitEfficiency` curve
`max(floor, fraction**exponent)` for GEMMs split into row chunks (medium
grained). SPEC.md:304 names the calibration hook: fit those parameters from
measured runs. This module holds the fitting arithmetic (pure Python, testable
on CPU) and writes the result in the reference's config schema
(`core/src/config.cpp:53-80` parse side, `:203-216` write side), so
`overlap-cli --config` could simulate with B200 numbers.

`scripts/calibrate_machine.py` takes the measurements on the GPU.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple


@dataclass
class SplitEfficiency:
    exponent: float = 0.15
    floor: float = 0.5

    def __call__(self, fraction: float) -> float:  # sim.cpp:47-50
        if fraction >= 1.0:
            return 1.0
        return max(self.floor, fraction ** self.exponent)


@dataclass
class MachineModel:
    """Field names, defaults and validation follow sim.hpp:25-42 / sim.cpp:52-57."""
    sm_count: int = 16
    flops_per_us: float = 2000.0
    launch_overhead_us: float = 20.0
    link_bw_bytes_per_us: float = 400.0
    link_latency_us: float = 2.0
    inter_node_bw_bytes_per_us: float = 0.0
    bytes_per_element: int = 8
    topology: Dict[str, object] = field(default_factory=lambda: {"kind": "NVLinkRing", "ranks_per_numa": 0,
                                                                  "ranks_per_node": 0})
    split_efficiency: SplitEfficiency = field(default_factory=SplitEfficiency)

    def validate(self) -> None:
        from ._native import ConfigError
        if self.sm_count <= 0 or self.flops_per_us <= 0 or self.link_bw_bytes_per_us <= 0 or self.bytes_per_element <= 0:
            raise ConfigError("machine rates and widths must be positive")
        if self.launch_overhead_us < 0 or self.link_latency_us < 0:
            raise ConfigError("machine overheads must be non-negative")

    def tile_time_us(self, tm: int, tn: int, local_k: int) -> float:  # sim.cpp:59-65
        return 2.0 * tm * tn * local_k / self.flops_per_us

    def gemm_nonsplit_us(self, tiles: int, tm: int, tn: int, local_k: int) -> float:  # sim.cpp:76-83
        waves = (tiles + self.sm_count - 1) // self.sm_count
        return self.launch_overhead_us + waves * self.tile_time_us(tm, tn, local_k)

    def to_json(self) -> Dict[str, object]:  # config.cpp:203-216 key order
        return {
            "sm_count": self.sm_count,
            "flops_per_us": self.flops_per_us,
            "launch_overhead_us": self.launch_overhead_us,
            "link_bw_bytes_per_us": self.link_bw_bytes_per_us,
            "link_latency_us": self.link_latency_us,
            "inter_node_bw_bytes_per_us": self.inter_node_bw_bytes_per_us,
            "bytes_per_element": self.bytes_per_element,
            "topology": dict(self.topology),
            "split_efficiency": {"exponent": self.split_efficiency.exponent, "floor": self.split_efficiency.floor},
        }


def linear_fit(xs: Sequence[float], ys: Sequence[float]) -> Tuple[float, float]:
    """Least squares y = a + b*x; returns (a, b)."""
    n = len(xs)
    if n < 2:
        raise ValueError("need at least two points")
    mx, my = sum(xs) / n, sum(ys) / n
    sxx = sum((x - mx) ** 2 for x in xs)
    if sxx == 0:
        raise ValueError("x values must not all be equal")
    b = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sxx
    return my - b * mx, b


def fit_compute(samples: Sequence[Tuple[int, float]], sm_count: int, tm: int, tn: int, local_k: int
                ) -> Tuple[float, float]:
    """samples: (tiles, measured GEMM microseconds) at one local_k. Fits the
    wave model t = L + ceil(tiles / sm_count) * tile_time and returns
    (launch_overhead_us, flops_per_us per slot)."""
    xs = [float((t + sm_count - 1) // sm_count) for t, _ in samples]
    ys = [us for _, us in samples]
    launch, tile_us = linear_fit(xs, ys)
    if tile_us <= 0:
        raise ValueError("non-positive tile time: measurements do not grow with the wave count")
    return max(0.0, launch), 2.0 * tm * tn * local_k / tile_us


def fit_link(samples: Sequence[Tuple[int, float]]) -> Tuple[float, float]:
    """samples: (bytes, microseconds) of single transfers. Fits t = latency +
    bytes / bw; returns (link_latency_us, link_bw_bytes_per_us)."""
    lat, inv_bw = linear_fit([float(b) for b, _ in samples], [us for _, us in samples])
    if inv_bw <= 0:
        raise ValueError("transfer time does not grow with size")
    return max(0.0, lat), 1.0 / inv_bw


def fit_split_efficiency(samples: Sequence[Tuple[float, float]]) -> SplitEfficiency:
    """samples: (chunk fraction f < 1, efficiency e = (t_full * f) / t_chunk).
    Least-squares exponent of e = f**x through the origin in log space; floor =
    the lowest efficiency observed (clamped to (0, 1])."""
    pts = [(f, e) for f, e in samples if 0.0 < f < 1.0 and e > 0.0]
    if not pts:
        raise ValueError("need chunk fractions in (0, 1)")
    num = sum(math.log(e) * math.log(f) for f, e in pts)
    den = sum(math.log(f) ** 2 for f, _ in pts)
    exponent = max(0.0, num / den)
    floor = min(1.0, max(1e-3, min(e for _, e in pts)))
    return SplitEfficiency(exponent=exponent, floor=floor)


def split_efficiency_samples(t_full_us: float, chunks: Dict[int, float]) -> List[Tuple[float, float]]:
    """chunks: partitions P -> measured time of one M/P chunk. Efficiency of a
    chunk relative to the full GEMM, as simulate_medium uses it (sim.cpp:463-468)."""
    return [(1.0 / p, (t_full_us / p) / t) for p, t in sorted(chunks.items()) if p > 1]


def reference_config(machine: MachineModel, problem: Dict[str, object], tile: Dict[str, int],
                     provenance: Dict[str, object]) -> Dict[str, object]:
    """A config in the reference's schema (configs/desk_machine_ag.json layout),
    with the calibration provenance alongside (ignored keys are rejected by the
    reference parser, so provenance lives in a separate top-level file field)."""
    machine.validate()
    return {
        "config": {
            "problem": problem,
            "tile": tile,
            "strategies": ["Coarse", "Medium", "Fine"],
            "machine": machine.to_json(),
            "run": {"swizzle": "RankShifted", "transfer": "Pull", "rows_per_comm_tile": tile["tm"]},
            "seed": 42,
        },
        "provenance": provenance,
    }
