"""GPU-calibrated autotuner over the reference's knob space.

Mirrors the reference tuner (core/src/tune.cpp, tune.hpp): the same knob
space (comm-tile halving `comm_tile_sizes` :23-34, `default_knob_space`
:51-65, cross-product `enumerate_knobs` :73-102 with ArrivalAligned skipped
on the scatter path), the same canonical encoding and tie-break on it
(:67-71, :225-233), the same cache file (`cache_key` = FNV-1a over problem,
machine, grid and objective, :114-127; JSON {cache_key, best_config,
objective_us}, :178-196, :237-243) and CSV/JSON reports (:247-276).

What changes on B200:
  * the objective is measured DEVICE time of the fused operator (CUDA events
    on its stream, L2 flushed before each repetition, median of >= 3 reps,
    dispersion (max-min)/median, noisy above 20 %) — the EngineWallClock
    analogue; the simulator objective is out of scope (no `sim`);
  * two B200 knobs join the grid: CTA group (1: 128x256 tiles, 2: CTA pairs
    with 256x256 tiles) and the AllGather transfer engine (1: copy engines,
    2: in-kernel TMA bulk copies);
  * every config is correctness-gated before its timing counts, like
    `verify_config` (:129-149): each rank's output is compared with an fp32
    cuBLAS product of the same bf16 operands on sampled rows; a mismatch aborts
    the whole pass naming the config.
"""
from __future__ import annotations

import json
import os
import statistics
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

from . import _native as N
from .comm import Communicator, ProblemSpec, TileShape

SWIZZLE_NAMES = {N.SWIZZLE_NAIVE: "Naive", N.SWIZZLE_RANK_SHIFTED: "RankShifted",
                 N.SWIZZLE_ARRIVAL_ALIGNED: "ArrivalAligned"}
TRANSFER_NAMES = {N.PULL: "Pull", N.PUSH: "Push"}
WRITE_NAMES = {N.WRITE_ALLTOALL: "WriteAlltoAll", N.FUSED_REDUCE: "FusedReduce"}
OBJECTIVES = ("DeviceTime",)


def comm_tile_sizes(rows_per_rank: int, tm: int) -> List[int]:
    """Successive halving from the row block down to the tile rows (tune.cpp:23-34)."""
    if tm <= 0 or rows_per_rank <= 0 or rows_per_rank % tm != 0:
        raise N.ConfigError("tile rows must divide rows per rank for comm tile halving")
    sizes = [rows_per_rank]
    v = rows_per_rank
    while v > tm and v % 2 == 0 and (v // 2) % tm == 0:
        v //= 2
        sizes.append(v)
    if sizes[-1] != tm:
        sizes.append(tm)
    return sizes


def _tile_fits(p: ProblemSpec, t: TileShape) -> bool:
    return t.tm > 0 and t.tn > 0 and p.rows_per_rank() % t.tm == 0 and p.local_cols() % t.tn == 0


def _largest_divisor_leq(value: int, cap: int) -> int:
    for d in range(min(value, cap), 0, -1):
        if value % d == 0:
            return d
    return 1


@dataclass
class KnobSpace:
    """tune.hpp:20-27 plus the B200 knobs (cta_groups, ag_engines)."""
    transfer_modes: List[int] = field(default_factory=list)
    swizzle_policies: List[int] = field(default_factory=list)
    gemm_tile_shapes: List[TileShape] = field(default_factory=list)
    write_modes: List[int] = field(default_factory=list)
    comm_tile_override: List[int] = field(default_factory=list)
    cta_groups: List[int] = field(default_factory=lambda: [0])
    ag_engines: List[int] = field(default_factory=lambda: [0])


def default_knob_space(problem: ProblemSpec, b200: bool = True) -> KnobSpace:
    """tune.cpp:51-65; with b200=True also CTA groups {1, 2} and AG engines {1, 2}."""
    ks = KnobSpace(transfer_modes=[N.PULL, N.PUSH],
                   swizzle_policies=[N.SWIZZLE_NAIVE, N.SWIZZLE_RANK_SHIFTED, N.SWIZZLE_ARRIVAL_ALIGNED],
                   write_modes=[N.WRITE_ALLTOALL, N.FUSED_REDUCE])
    for t in (TileShape(64, 64), TileShape(128, 64), TileShape(64, 128), TileShape(128, 128)):
        if _tile_fits(problem, t):
            ks.gemm_tile_shapes.append(t)
    if not ks.gemm_tile_shapes:
        ks.gemm_tile_shapes.append(TileShape(_largest_divisor_leq(problem.rows_per_rank(), 64),
                                             _largest_divisor_leq(problem.local_cols(), 64)))
    if b200:
        ks.cta_groups = [1, 2]
        ks.ag_engines = [1, 2] if problem.pattern == N.ALLGATHER_GEMM and problem.local_k() % 8 == 0 else [0]
    return ks


@dataclass(frozen=True)
class TuneConfig:
    """tune.hpp:29-37; `encode` is the reference string plus the B200 knobs
    when they are not automatic."""
    tile: TileShape
    swizzle: int = N.SWIZZLE_NAIVE
    rows_per_comm_tile: int = 0
    transfer: int = N.PULL
    write: int = N.FUSED_REDUCE
    cta_group: int = 0
    ag_engine: int = 0

    def encode(self) -> str:
        s = (f"tile={self.tile.tm}x{self.tile.tn};comm={self.rows_per_comm_tile};"
             f"swizzle={SWIZZLE_NAMES[self.swizzle]};transfer={TRANSFER_NAMES[self.transfer]};"
             f"write={WRITE_NAMES[self.write]}")
        if self.cta_group:
            s += f";cta={self.cta_group}"
        if self.ag_engine:
            s += f";engine={'copy' if self.ag_engine == 1 else 'sm'}"
        return s


def enumerate_knobs(problem: ProblemSpec, knobs: KnobSpace) -> List[TuneConfig]:
    """Cross product in the reference's order (tune.cpp:73-102), B200 knobs innermost."""
    problem.validate()
    grid: List[TuneConfig] = []
    for tile in knobs.gemm_tile_shapes:
        if not _tile_fits(problem, tile):
            continue
        if knobs.comm_tile_override:
            comms = [c for c in knobs.comm_tile_override if c > 0 and problem.rows_per_rank() % c == 0]
        else:
            comms = comm_tile_sizes(problem.rows_per_rank(), tile.tm)
        if problem.pattern == N.ALLGATHER_GEMM:
            for tm in knobs.transfer_modes:
                for c in comms:
                    for sw in knobs.swizzle_policies:
                        for cg in knobs.cta_groups:
                            for eng in knobs.ag_engines:
                                grid.append(TuneConfig(tile, sw, c, tm, N.FUSED_REDUCE, cg, eng))
        else:
            for wm in knobs.write_modes:
                for sw in knobs.swizzle_policies:
                    if sw == N.SWIZZLE_ARRIVAL_ALIGNED:
                        continue  # arrival alignment is an AllGather-side policy
                    for cg in knobs.cta_groups:
                        grid.append(TuneConfig(tile, sw, problem.rows_per_rank(), N.PULL, wm, cg, 0))
    if not grid:
        raise N.ConfigError("empty knob space for this problem")
    return grid


def fnv1a(s: str, h: int = 1469598103934665603) -> int:
    for ch in s.encode():
        h ^= ch
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def cache_key_for(problem: ProblemSpec, machine: str, grid: Sequence[TuneConfig], objective: str) -> str:
    """tune.cpp:114-127 with the machine model replaced by the measured device."""
    pat = "AllGatherGemm" if problem.pattern == N.ALLGATHER_GEMM else "GemmReduceScatter"
    blob = f"{pat},{problem.m},{problem.n},{problem.k},{problem.tp}|{machine}|{objective}"
    for c in grid:
        blob += "|" + c.encode()
    return f"{fnv1a(blob):016x}"


@dataclass
class TuneEntry:
    config: TuneConfig
    objective_us: float = 0.0
    repetitions: int = 1
    dispersion: float = 0.0
    noisy: bool = False


@dataclass
class TuneResult:
    best_config: Optional[TuneConfig] = None
    objective_us: float = 0.0
    table: List[TuneEntry] = field(default_factory=list)
    from_cache: bool = False
    cache_key: str = ""


def tune(problem: ProblemSpec, knobs: KnobSpace, measure: Callable[[TuneConfig], List[float]],
         verify: Callable[[TuneConfig], None], objective: str = "DeviceTime", repetitions: int = 5,
         cache_path: str = "", machine: str = "") -> TuneResult:
    """tune.cpp:169-245. `verify(cfg)` raises on a wrong result; `measure(cfg)`
    returns `repetitions` objective samples in microseconds."""
    if objective not in OBJECTIVES:
        raise N.ConfigError(f"unknown objective: '{objective}' (expected DeviceTime)")
    if repetitions < 3:
        raise N.ConfigError("device-time objective requires repetitions >= 3")
    grid = enumerate_knobs(problem, knobs)
    key = cache_key_for(problem, machine, grid, objective)
    if cache_path and os.path.exists(cache_path):
        with open(cache_path) as f:
            j = json.load(f)
        if j.get("cache_key", "") == key:
            for c in grid:
                if c.encode() == j["best_config"]:
                    return TuneResult(best_config=c, objective_us=float(j["objective_us"]), from_cache=True,
                                      cache_key=key)
    result = TuneResult(cache_key=key)
    for cfg in grid:
        try:
            verify(cfg)
        except Exception as e:
            raise RuntimeError(f"tuning aborted: config [{cfg.encode()}] failed verification: {e}") from e
        samples = sorted(measure(cfg))
        med = samples[len(samples) // 2]
        disp = (samples[-1] - samples[0]) / med if med > 0 else 0.0
        result.table.append(TuneEntry(cfg, med, len(samples), disp, disp > 0.20))
    best = min(result.table, key=lambda e: (e.objective_us, e.config.encode()))
    result.best_config, result.objective_us = best.config, best.objective_us
    if cache_path:
        with open(cache_path, "w") as f:
            f.write(json.dumps({"cache_key": key, "best_config": best.config.encode(),
                                "objective_us": best.objective_us}, indent=2) + "\n")
    return result


def write_tune_csv(path: str, result: TuneResult) -> None:
    """tune.cpp:247-259."""
    best = result.best_config.encode()
    with open(path, "w") as f:
        f.write("config,objective_us,repetitions,dispersion,noisy,best\n")
        for e in result.table:
            f.write(f"{e.config.encode()},{e.objective_us:.6f},{e.repetitions},{e.dispersion:.4f},"
                    f"{int(e.noisy)},{int(e.config.encode() == best)}\n")


def write_tune_json(path: str, result: TuneResult) -> None:
    """tune.cpp:261-276."""
    j = {"best_config": result.best_config.encode(), "objective_us": result.objective_us,
         "from_cache": result.from_cache, "cache_key": result.cache_key,
         "table": [{"config": e.config.encode(), "objective_us": e.objective_us, "repetitions": e.repetitions,
                    "dispersion": e.dispersion, "noisy": e.noisy} for e in result.table]}
    with open(path, "w") as f:
        f.write(json.dumps(j, indent=2) + "\n")


# ---------------------------------------------------------------------------
# GPU objective and correctness gate on a communicator whose library buffers
# hold the inputs (every rank's A and B shard), all ranks on this process.
# ---------------------------------------------------------------------------
def machine_id(device: int = 0) -> str:
    import torch

    prop = torch.cuda.get_device_properties(device)
    return f"{prop.name},{prop.multi_processor_count}"


def run_config(comm: Communicator, problem: ProblemSpec, cfg: TuneConfig, streams=None, opts=None) -> None:
    o = opts if opts is not None else N.default_opts()
    o.cta_group, o.ag_engine = cfg.cta_group, cfg.ag_engine
    swizzle = cfg.swizzle != N.SWIZZLE_NAIVE
    if problem.pattern == N.ALLGATHER_GEMM:
        comm.ag_gemm(problem, cfg.tile, cfg.rows_per_comm_tile, cfg.transfer, swizzle, o, streams)
    else:
        o.deterministic_reduce = 1 if cfg.write == N.WRITE_ALLTOALL else 0
        comm.gemm_rs(problem, cfg.tile, cfg.write, swizzle, o, streams)


def gpu_measure(comm: Communicator, problem: ProblemSpec, repetitions: int, streams=None):
    """Device time (us) of the operator per repetition: CUDA events on its
    stream, 256 MiB written between repetitions to flush the 126 MB L2."""
    import torch

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    if streams is None:
        streams = [stream.cuda_stream] * len([r for r in range(problem.tp)])

    def measure(cfg: TuneConfig) -> List[float]:
        run_config(comm, problem, cfg, streams)  # warm-up (schedules uploaded, clocks up)
        comm.sync()
        out = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(repetitions):
            flush.zero_()
            e0.record(stream)
            run_config(comm, problem, cfg, streams)
            e1.record(stream)
            e1.synchronize()
            out.append(e0.elapsed_time(e1) * 1e3)
        comm.sync()
        return out

    return measure


def gpu_verify(comm: Communicator, problem: ProblemSpec, rows: int = 64, tol: float = 8e-3, streams=None):
    """Correctness gate (the reference's verify_config, tune.cpp:129-149): each
    rank's bf16 output on `rows` sampled rows against the fp64 product of the
    same bf16 operands (the oracle's definition: k-ascending fp64 GEMM, RS
    partials summed in rank order), with the reference metric max|a-b| /
    max(1, |a|, |b|) (matrix.cpp:11-25) and the stated bf16 tolerance."""
    import torch

    tp = problem.tp
    a = [comm.tensor(r, N.BUF_A_SHARD, problem).double() for r in range(tp)]
    b = [comm.tensor(r, N.BUF_B_SHARD, problem).double() for r in range(tp)]
    dev = a[0].device
    m_out = problem.m if problem.pattern == N.ALLGATHER_GEMM else problem.rows_per_rank()
    idx = torch.linspace(0, m_out - 1, steps=min(rows, m_out), device=dev).round().long().unique()
    if problem.pattern == N.ALLGATHER_GEMM:
        gathered = torch.cat([x.to(dev) for x in a])[idx]
        refs = [gathered.to(b[r].device) @ b[r].t() for r in range(tp)]
    else:
        rpr = problem.rows_per_rank()
        refs = []
        for r in range(tp):
            rows_g = idx + r * rpr
            acc = None
            for s in range(tp):  # rank order, like the oracle's reduce (oracle.cpp:49-53)
                part = (a[s][rows_g.to(a[s].device)] @ b[s].t()).to(dev)
                acc = part if acc is None else acc + part
            refs.append(acc)

    def verify(cfg: TuneConfig) -> None:
        run_config(comm, problem, cfg, streams)
        comm.sync()
        for r in range(tp):
            got = comm.tensor(r, N.BUF_C_OUT, problem).double()
            ref = refs[r].to(got.device)
            got = got[idx.to(got.device)]
            den = torch.maximum(torch.maximum(got.abs(), ref.abs()), torch.ones_like(ref))
            err = ((got - ref).abs() / den).max().item()
            if not err <= tol:
                raise AssertionError(f"rank {r}: max rel err {err:.3e} > {tol}")

    return verify
