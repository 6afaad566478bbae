"""Benchmark of the fused tensor-parallel operators (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload llama70b-up-ag|llama70b-down-rs|gpt3-ag|gpt3-rs]

A step is one fused operator over the whole workload. N=1: all TP ranks of
the workload are emulated on cuda:0 (one fused launch covering every rank,
copy-engine transfers between the ranks' symmetric heaps). N>1 (torchrun): one
process per GPU, TP = N over cudaIpc-mapped heaps (NVLink), the same global
GEMM (strong scaling). Prints ONE JSON line on rank 0.

`--impl reference` times the reference's own CPU engine (oracle/_ref, compiled
from /root/reference; oracle port if absent) on a bounded sample of the same
workload, on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused AG-GEMM/GEMM-RS TFLOPS + comm-overlap % at TP=2/4/8 vs cuBLAS+NCCL"

WORKLOADS = {
    # name: (pattern, m, n, k, tp, description)  — BASELINE.json configs[1..3]
    "llama70b-up-ag": (0, 4096, 28672, 8192, 8, "AllGather-GEMM Llama-2-70B MLP up-proj (M=4096, K=8192, N=28672) bf16"),
    "llama70b-down-rs": (1, 4096, 8192, 28672, 8, "GEMM-ReduceScatter Llama-2-70B MLP down-proj (M=4096, K=28672, N=8192) bf16"),
    "gpt3-ag": (0, 8192, 49152, 12288, 8, "AllGather-GEMM GPT-3 175B MLP (M=8192, K=12288, N=49152) bf16"),
    "gpt3-rs": (1, 8192, 12288, 49152, 8, "GEMM-ReduceScatter GPT-3 175B MLP (M=8192, K=49152, N=12288) bf16"),
    "llama70b-down-rs-tp4": (1, 4096, 8192, 28672, 4, "GEMM-ReduceScatter Llama-2-70B MLP down-proj at TP=4 (M=4096, K=28672, N=8192) bf16"),
    "llama70b-down-rs-tp2": (1, 4096, 8192, 28672, 2, "GEMM-ReduceScatter Llama-2-70B MLP down-proj at TP=2 (M=4096, K=28672, N=8192) bf16"),
    "rs-1024-tp2": (1, 1024, 1024, 1024, 2, "GEMM-ReduceScatter M=N=K=1024 at TP=2 (oracle plumbing config)"),
    # BASELINE.json configs[4] (decode sweep) representatives; scripts/decode_sweep.py runs the full sweep
    "decode-ag-up-m16": (0, 16, 28672, 8192, 8, "decode AllGather-GEMM Llama-2-70B MLP up-proj, M=16 tokens, TP=8"),
    "decode-rs-down-m16": (1, 16, 8192, 28672, 8, "decode GEMM-ReduceScatter Llama-2-70B MLP down-proj, M=16, TP=8"),
    "decode-rs-attn-m16": (1, 16, 8192, 8192, 8, "decode GEMM-ReduceScatter Llama-2-70B attention-out, M=16, TP=8"),
    "decode-ag-up-m128": (0, 128, 28672, 8192, 8, "decode AllGather-GEMM Llama-2-70B MLP up-proj, M=128 tokens, TP=8"),
    "decode-ag-up-m256": (0, 256, 28672, 8192, 8, "decode AllGather-GEMM Llama-2-70B MLP up-proj, M=256 tokens, TP=8"),
    "decode-ag-up-m512": (0, 512, 28672, 8192, 8, "decode AllGather-GEMM Llama-2-70B MLP up-proj, M=512 tokens, TP=8"),
    "decode-rs-down-m256": (1, 256, 8192, 28672, 8, "decode GEMM-ReduceScatter Llama-2-70B MLP down-proj, M=256, TP=8"),
    "decode-rs-down-m512": (1, 512, 8192, 28672, 8, "decode GEMM-ReduceScatter Llama-2-70B MLP down-proj, M=512, TP=8"),
    "decode-rs-attn-m128": (1, 128, 8192, 8192, 8, "decode GEMM-ReduceScatter Llama-2-70B attention-out, M=128, TP=8"),
    "decode-rs-attn-m512": (1, 512, 8192, 8192, 8, "decode GEMM-ReduceScatter Llama-2-70B attention-out, M=512, TP=8"),
    # One GPU's share of configs[4] at real TP=8 (per-GPU decode vs the ~9 us HBM roofline):
    # the per-rank GEMM shapes as TP=1 problems (the rank's weight shard streamed once).
    "rank-decode-ag-up-m16": (0, 16, 3584, 8192, 1, "one rank of decode AG-GEMM Llama-2-70B up-proj at TP=8: M=16, K=8192, N/TP=3584 (58.7 MB weight shard)"),
    "rank-decode-ag-up-m128": (0, 128, 3584, 8192, 1, "one rank of decode AG-GEMM Llama-2-70B up-proj at TP=8: M=128, K=8192, N/TP=3584"),
    "rank-decode-rs-down-m16": (1, 16, 8192, 3584, 1, "one rank of decode GEMM-RS Llama-2-70B down-proj at TP=8: M=16, K/TP=3584, N=8192 (58.7 MB weight shard)"),
    "rank-decode-rs-down-m128": (1, 128, 8192, 3584, 1, "one rank of decode GEMM-RS Llama-2-70B down-proj at TP=8: M=128, K/TP=3584, N=8192"),
    "rank-decode-rs-attn-m16": (1, 16, 8192, 1024, 1, "one rank of decode GEMM-RS Llama-2-70B attention-out at TP=8: M=16, K/TP=1024, N=8192 (16.8 MB weight shard)"),
}
NVLINK_GBS = 900.0  # NVLink 5 per direction per GPU (B200_PROFILING.md)
FALLBACK_PEAKS = {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_PEAKS, "fallback (B200_PROFILING.md)"


def roofline_work(pattern, m, n, k, tp, emulated, partial_bytes=4):
    """Algorithmic work of ONE fused launch: (flops, HBM bytes,
    NVLink bytes). Per rank:
      AG  flops 2·M·(N/TP)·K; NVLink ingress (TP−1)/TP·M·K·2; HBM a_agg write +
          read 2·M·K·2 + weight K·(N/TP)·2 + C M·(N/TP)·2 + the shard rows this
          GPU serves its peers (TP−1)/TP·M·K·2.
      RS  flops 2·M·N·(K/TP); NVLink egress (TP−1)/TP·M·N·4 (fp32 partials);
          HBM A M·(K/TP)·2 + weight (K/TP)·N·2 + partials written by / read
          for the owners 2·(TP−1)/TP·M·N·4 + C (M/TP)·N·2.
    N=1 (every rank emulated on one GPU, one launch): TP × the per-rank work,
    the transfers are HBM traffic (no NVLink term). N>1: one rank's work."""
    rpr = m // tp
    if pattern == 0:
        nl = n // tp
        flops = 2.0 * m * nl * k
        nvl = (tp - 1) / tp * m * k * 2
        hbm = 2.0 * m * k * 2 + k * nl * 2 + m * nl * 2 + nvl
    else:
        kl = k // tp
        flops = 2.0 * m * n * kl
        nvl = (tp - 1) / tp * m * n * partial_bytes
        hbm = m * kl * 2.0 + kl * n * 2 + 2 * nvl + rpr * n * 2
    ranks = tp if emulated else 1
    return flops * ranks, hbm * ranks, (0.0 if emulated else nvl)


def roofline_of(work, kernel_ms, pk, src):
    """The bound is the slowest of tensor-core time, HBM time and NVLink time
    at peak (north_star: "the slower of the compute at peak and the bytes over
    NVLink", plus HBM so decode fractions stay <= 1); achieved and peak are in
    the bound's unit, frac = roofline time / measured kernel time."""
    flops, hbm, nvl = work
    terms = {"tensor": flops / (pk["bf16_tflops"] * 1e12), "hbm": hbm / (pk["hbm_gbs"] * 1e9),
             "nvlink": nvl / (NVLINK_GBS * 1e9)}
    bound = max(terms, key=terms.get)
    t = kernel_ms * 1e-3
    if bound == "tensor":
        achieved, peak, unit = flops / t / 1e12, pk["bf16_tflops"], "TFLOP/s"
    elif bound == "hbm":
        achieved, peak, unit = hbm / t / 1e9, pk["hbm_gbs"], "GB/s"
    else:
        achieved, peak, unit = nvl / t / 1e9, NVLINK_GBS, "GB/s"
    return {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
            "terms_us": {k2: v * 1e6 for k2, v in terms.items()}, "roofline_us": terms[bound] * 1e6,
            "kernel_ms": kernel_ms, "flops_per_launch": flops, "hbm_bytes_per_launch": hbm,
            "nvlink_bytes_per_launch": nvl,
            "peak_source": f"{src}: burst bf16 {pk['bf16_tflops']} TFLOP/s, HBM {pk['hbm_gbs']} GB/s; "
                           f"NVLink {NVLINK_GBS} GB/s per direction (nominal)"}


def bf16_tol(k):
    """Parity tolerance for bf16 outputs (oracle/gpu_harness.tol):
    8e-3 plus the fp32 accumulation term beyond k = 32768."""
    return 8e-3 + max(0.0, 1e-4 * max(1.0, k / 1024.0) - 3.2e-3)


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference engine (or the oracle port) on a bounded sample
# ---------------------------------------------------------------------------
def cpu_sample_shape(pattern, m, n, k, tp):
    """Bounded sample of the workload: the same K/N (and TP), M cut to 8 rows per rank."""
    ms = 8 * tp
    return ms, n, k


def run_cpu_reference(pattern, m, n, k, tp, reps=1):
    """Times the reference's fused engine on the host cores; returns the
    cpu_baseline object (TFLOPS over the sample)."""
    from oracle import oracle as O

    ms, ns, ks = cpu_sample_shape(pattern, m, n, k, tp)
    cores = os.cpu_count() or 1
    flops = 2.0 * ms * ns * ks
    times = []
    if O.ref_available():
        workers = max(1, cores // tp)
        tn = 256 if (ns // tp if pattern == 0 else ns) % 256 == 0 else 1
        which = O.FUSED_AG if pattern == 0 else O.FUSED_RS
        for _ in range(reps):
            secs, _ = O.ref_run(which, pattern, ms, ns, ks, tp, 42, True, tm=8, tn=tn, rpct=8, transfer=0,
                                write_mode=0, swizzle=True, workers=workers, want_outputs=False)
            times.append(secs)
        kind, used = "reference", tp * workers + (tp if pattern == 0 else tp)
        what = (f"reference {'run_fused_allgather_gemm (Pull, swizzle)' if pattern == 0 else 'run_fused_gemm_reducescatter (WriteAlltoAll, swizzle)'}"
                f" fp64, oracle/_ref built from /root/reference, {workers} workers/rank + 1 transfer/reduce agent per rank"
                f" = {tp * workers + tp} threads")
    else:
        import numpy as np

        for _ in range(reps):
            a, b = zip(*[O.rank_inputs(pattern, ms, ns, ks, tp, 42, r, True) for r in range(tp)])
            t0 = time.perf_counter()
            O.dense_oracle(pattern, ms, ns, ks, tp, a, b)
            times.append(time.perf_counter() - t0)
            del np
        kind, used = "port", 1
        what = "oracle port (oracle/flux_oracle.c dense fp64 restatement, 1 thread)"
    t = statistics.median(times)
    return {"value": flops / t / 1e12, "unit": "TFLOPS", "cores": used, "kind": kind,
            "sample": f"{what}; M={ms} (8 rows/rank), N={ns}, K={ks}, TP={tp}; {flops / 1e9:.1f} GFLOP per run; "
                      f"median of {len(times)} run(s) = {t:.2f} s; host has {cores} cores"}


def reference_arm(args, wl):
    pattern, m, n, k, tp, desc = WORKLOADS[wl]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        tp = world  # the same TP = N problem as our arm's N>1 run
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    base = None
    for _ in range(args.warmup):
        run_cpu_reference(pattern, m, n, k, tp, reps=1)
    vals = []
    ms, ns, ks = cpu_sample_shape(pattern, m, n, k, tp)
    for _ in range(args.steps):
        base = run_cpu_reference(pattern, m, n, k, tp, reps=1)
        vals.append(base["value"])
    v = statistics.median(vals)
    base["value"] = v
    ms_step = 2.0 * ms * ns * ks / (v * 1e12) * 1e3  # one bounded sample (sample_m rows) per step
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOPS", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference Rng stream)",
            "config": {"workload": wl, "description": desc, "m": m, "n": n, "k": k, "tp": tp,
                       "sample_m": cpu_sample_shape(pattern, m, n, k, tp)[0]},
            "cpu_baseline": base,
            "e2e": {"value": v, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def our_arm(args, wl):
    import ctypes as C

    import torch

    import paper_2406_06858_b200 as fx
    from paper_2406_06858_b200 import _native as N
    from paper_2406_06858_b200 import baselines as BL

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    # FLUX_BENCH_SHARE_GPU=1 (tests only): every rank on the visible GPUs modulo
    # their count, gloo for the plumbing — runs the N>1 (IPC) path on a one-GPU box.
    share = os.environ.get("FLUX_BENCH_SHARE_GPU") == "1"
    if share:
        local_rank = local_rank % max(1, torch.cuda.device_count())
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    # A real (non-legacy) stream: the library runs on it and the CUDA events
    # below are recorded on it.
    torch.cuda.set_stream(torch.cuda.Stream(device=dev))

    pattern, m, n, k, tp_wl, desc = WORKLOADS[wl]
    emulated = world == 1
    tp = tp_wl if emulated else world
    prob = fx.ProblemSpec(m, n, k, tp, pattern)
    heap = fx.required_heap_bytes(prob) + (64 << 20)
    # --nvls: NVLS multicast (the AllGather push / GEMM-RS owner sums through the
    # NVSwitch); ranks emulated on one GPU run the same protocol with unicast
    # loops (FLUX_NVLS_EMULATED). Off by default; "unavailable" (with the reason)
    # when the host exposes no multicast, and the run continues without it.
    nvls_mode, nvls_note = fx.NVLS_OFF, None
    if emulated:
        comm = fx.Communicator(tp, [local_rank] * tp, heap_bytes=heap)
        my_ranks = list(range(tp))
        if args.nvls:
            nvls_mode, nvls_note = fx.NVLS_EMULATED, "emulated (unicast loops over the ranks' regions on one GPU)"
    else:
        def gather(blob):
            out = [None] * world
            dist.all_gather_object(out, blob)
            return out
        comm = None
        if args.nvls:
            try:
                comm = fx.Communicator.ipc(rank, tp, local_rank, heap, gather, nvls_bytes=fx.nvls_required_bytes(prob))
                nvls_mode, nvls_note = fx.NVLS_MULTICAST, "multicast (multimem through the NVSwitch)"
            except fx.FluxError as e:
                nvls_note = "unavailable: " + str(e)
        if comm is None:
            comm = fx.Communicator.ipc(rank, tp, local_rank, heap, gather)
        my_ranks = [rank]

    # synthetic inputs (uniform [-1, 1), bf16) straight into the symmetric heaps
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    for r in my_ranks:
        for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
            t = comm.tensor(r, kind, prob)
            t.copy_(torch.rand(t.shape, generator=g, device=dev).mul_(2).sub_(1))
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream().cuda_stream
    streams = [stream] * (tp if emulated else 1)
    tile = fx.TileShape(prob.rows_per_rank(), prob.local_cols())
    opts = fx.default_opts(ag_engine=args.ag_engine, cta_group=args.cta_group,
                           deterministic_reduce=0 if args.nondeterministic else 1, nvls=nvls_mode)
    # L2 flush between timed steps (outside the events): write 256 MiB (> the
    # 126 MB L2), then read another 256 MiB so the written lines are evicted
    # (written back) before the next step starts — no dirty lines are left to
    # drain inside the timed region.
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_rd = torch.ones(64 << 20, dtype=torch.int32, device=dev)

    def l2_flush():
        flush.zero_()
        flush_rd.max()

    def op():
        if pattern == 0:
            comm.ag_gemm(prob, tile, prob.rows_per_rank(), fx.PULL, True, opts, streams)
        else:
            comm.gemm_rs(prob, tile, args.write_mode, True, opts, streams)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps, warmup, kernel_times=None):
        """Sum of per-step device times (CUDA events on the launch stream), L2
        flushed between steps outside the timed events; max over ranks."""
        for _ in range(warmup):
            fn()
        barrier()
        total = 0.0
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(steps):
            l2_flush()
            ev0.record()
            fn()
            ev1.record()
            ev1.synchronize()
            total += ev0.elapsed_time(ev1)
            if kernel_times is not None:
                kernel_times.append(comm.last_kernel_ms())
        barrier()
        t = torch.tensor([total], device=dev)
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item() / steps

    def interleaved(fns, rounds):
        """Per-variant median device time (max over ranks), one step of every
        variant per round."""
        for fn in fns.values():
            fn()
            fn()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        times = {name: [] for name in fns}
        for _ in range(rounds):
            for name, fn in fns.items():
                l2_flush()
                barrier()
                ev0.record()
                fn()
                ev1.record()
                ev1.synchronize()
                times[name].append(ev0.elapsed_time(ev1))
        barrier()
        out = {}
        for name, ts in times.items():
            t = torch.tensor([statistics.median(ts)], device=dev)
            if dist is not None:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            out[name] = t.item()
        return out

    def parity_check():
        """Row-sampled check of every rank's output of the last timed step
        against an fp64 product of the same bf16 inputs (the oracle's math,
        k-ascending dense dot products, rank-ordered sums; SURVEY §8c option
        iii): a few rows per ownership block (first, last, comm-tile edges),
        every column. At N>1 the sampled A rows / partial rows are exchanged
        with torch.distributed, so a multi-GPU run checks itself."""
        tp_ = prob.tp
        rpr = prob.rows_per_rank()
        offs = sorted({0, rpr - 1, rpr // 2, min(rpr - 1, 127), min(rpr - 1, 128)})
        rows = [o * rpr + j for o in range(tp_) for j in offs]
        S = len(rows)
        idx = torch.tensor(rows, device=dev)
        cpu_coll = dist is not None and share  # gloo plumbing: collectives on host tensors

        def allsum(t):
            if dist is None:
                return t
            if cpu_coll:
                h = t.cpu()
                dist.all_reduce(h)
                return h.to(dev)
            dist.all_reduce(t)
            return t

        worst = 0.0
        if pattern == 0:
            a_rows = torch.zeros(S, prob.local_k(), dtype=torch.float64, device=dev)
            for i, gr in enumerate(rows):
                o = gr // rpr
                if o in my_ranks:
                    a_rows[i] = comm.tensor(o, N.BUF_A_SHARD, prob)[gr - o * rpr].double()
            a_rows = allsum(a_rows)
            for r in my_ranks:
                want = a_rows @ comm.tensor(r, N.BUF_B_SHARD, prob).double().t()
                got = comm.tensor(r, N.BUF_C_OUT, prob).index_select(0, idx).double()
                err = ((got - want).abs() / torch.clamp(torch.maximum(got.abs(), want.abs()), min=1.0)).max().item()
                worst = max(worst, err)
        else:
            part = torch.zeros(S, prob.n, dtype=torch.float64, device=dev)
            for r in my_ranks:  # rank order on one process (emulated); all_reduce across processes
                a_s = comm.tensor(r, N.BUF_A_SHARD, prob).index_select(0, idx).double()
                part += a_s @ comm.tensor(r, N.BUF_B_SHARD, prob).double().t()
            part = allsum(part)
            for r in my_ranks:
                sel = [i for i, gr in enumerate(rows) if gr // rpr == r]
                local = torch.tensor([rows[i] - r * rpr for i in sel], device=dev)
                got = comm.tensor(r, N.BUF_C_OUT, prob).index_select(0, local).double()
                want = part[sel]
                err = ((got - want).abs() / torch.clamp(torch.maximum(got.abs(), want.abs()), min=1.0)).max().item()
                worst = max(worst, err)
        t = torch.tensor([worst], device=dev)
        if dist is not None:
            if cpu_coll:
                t = t.cpu()
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        worst = t.item()
        tol = bf16_tol(prob.local_k())
        return {"rows_checked_per_rank": S if pattern == 0 else len(offs), "max_rel_error": worst, "tol": tol,
                "pass": bool(worst <= tol),
                "reference": "fp64 product of the sampled rows on the same bf16 inputs (max_rel_error, "
                             "matrix.cpp:11-25), max over ranks"}

    ag_transfer = ("copy-engine pull" if N.lib().flux_ag_engine(C.byref(prob.c()), fx.PULL, C.byref(opts)) == 1
                   else "in-kernel TMA pull (the GEMM's SMs)")

    # ---- headline: the fused operator ----
    comm.set_timing(True)
    kernel_ms = []
    with ClockSampler(local_rank) as clk:
        ms_fused = timed(op, args.steps, max(3, args.warmup), kernel_ms)
    comm.sync()
    launches_per_step = comm.last_launch_count()
    comm.set_timing(False)
    flops = prob.flops()
    value = flops / (ms_fused * 1e-3) / 1e12
    parity = parity_check()

    # ---- Eq. 1 / Eq. 2 ingredients ----
    # Measured round-robin (one step of each variant per round, L2 flushed
    # before each, medians over the rounds) so clock / power drift during the
    # run biases no variant; the fused op is re-measured in the same rounds.
    extra = {}
    if not args.quick:
        # cuBLAS + NCCL (or device copies when emulated): B1, and cuBLAS non-split GEMM
        if emulated:
            if pattern == 0:
                shards = [comm.tensor(r, N.BUF_A_SHARD, prob).contiguous() for r in range(tp)]
                weights = [comm.tensor(r, N.BUF_B_SHARD, prob).contiguous() for r in range(tp)]
                b = BL.EmulatedAG(shards, weights)
            else:
                a_s = [comm.tensor(r, N.BUF_A_SHARD, prob).contiguous() for r in range(tp)]
                w_s = [comm.tensor(r, N.BUF_B_SHARD, prob).contiguous() for r in range(tp)]
                b = BL.EmulatedRS(a_s, w_s)
        else:
            if pattern == 0:
                b = BL.DistAG(comm.tensor(rank, N.BUF_A_SHARD, prob).contiguous(),
                              comm.tensor(rank, N.BUF_B_SHARD, prob).contiguous(), host_collectives=share)
            else:
                b = BL.DistRS(comm.tensor(rank, N.BUF_A_SHARD, prob).contiguous(),
                              comm.tensor(rank, N.BUF_B_SHARD, prob).contiguous(), host_collectives=share)
        if pattern == 0:
            b.unfused()  # fills the gathered buffers for gemm_only
        variants = {"fused": op, "local": lambda: comm.local_gemm(prob, opts, streams),
                    "nonoverlap": lambda: comm.nonoverlap(prob, opts, streams),
                    "cublas_gemm": b.gemm_only, "b1": b.unfused}
        if (emulated and pattern == 0) or not emulated:
            variants["b2"] = b.decomposed  # cuBLAS chunk GEMMs + chunked copies / NCCL (run_medium_grained)
        if emulated:  # the device decomposed baseline (flux_medium_grained, tp chunks)
            tile_b2 = fx.TileShape(prob.rows_per_rank(), prob.local_cols())
            variants["b2_ours"] = lambda: comm.medium_grained(prob, tile_b2, tp, opts, streams)
        med = interleaved(variants, max(5, args.steps // 2))
        del b
        ms_f = med["fused"]
        t_gemm = min(med["local"], med["cublas_gemm"])
        # Eq. 2 (sim.cpp:577-586): ECT = T_op - T_gemm_nonsplit, E = 1 - ECT_fused / ECT_unfused. Each
        # operator's exposed communication is taken against ITS OWN GEMM (the fused op against our
        # plain GEMM, B1 against cuBLAS), so neither GEMM's speed counts as communication.
        ect_fused = ms_f - med["local"]
        ect_b1 = med["b1"] - med["cublas_gemm"]
        # Second form: against our own serial baseline (run_nonoverlap: the same GEMM kernel after a
        # serial copy-engine AllGather / before a serial reduce) — the same GEMM on both sides.
        ect_serial = med["nonoverlap"] - med["local"]
        extra = {
            "t_fused_ms": ms_f, "t_gemm_nonsplit_ms": t_gemm, "t_gemm_ours_ms": med["local"],
            "t_gemm_cublas_ms": med["cublas_gemm"], "t_unfused_cublas_ms": med["b1"], "t_decomposed_ms": med.get("b2"),
            "t_decomposed_ours_ms": med.get("b2_ours"),
            "t_nonoverlap_ours_ms": med["nonoverlap"],
            "ect_fused_ms": ect_fused, "ect_unfused_ms": ect_b1, "ect_nonoverlap_ours_ms": ect_serial,
            "overlap_efficiency": (1.0 - ect_fused / ect_b1) if ect_b1 > 0 else None,
            "overlap_efficiency_vs_our_serial": (1.0 - ect_fused / ect_serial) if ect_serial > 0 else None,
            "speedup_vs_unfused": med["b1"] / ms_f,
            "speedup_vs_decomposed": (med["b2"] / ms_f) if med.get("b2") else None,
            "speedup_vs_our_serial": med["nonoverlap"] / ms_f,
            "method": "round-robin medians (one step of each variant per round, L2 flushed before each); "
                      "ECT of each operator against its own GEMM (fused: our plain GEMM; B1: cuBLAS)",
            "unfused_baseline": ("device copies + cuBLAS (ranks emulated on one GPU)" if emulated
                                 else ("gloo host collectives + cuBLAS (ranks sharing one GPU, test plumbing)" if share
                                       else "NCCL + cuBLAS")),
            "decomposed_baseline": ("cuBLAS chunk GEMMs + side-stream device copies" if emulated
                                    else "cuBLAS chunk GEMMs + per-chunk NCCL broadcast / reduce (async)"),
        }

    # ---- e2e through the C ABI with host buffers ----
    e2e = None
    if not args.quick:
        a_host = {r: torch.empty(prob.rows_per_rank() if pattern == 0 else m, prob.local_k(), dtype=torch.bfloat16,
                                 pin_memory=True) for r in my_ranks}
        c_rows = m if pattern == 0 else prob.rows_per_rank()
        c_host = {r: torch.empty(c_rows, prob.local_cols(), dtype=torch.bfloat16, pin_memory=True) for r in my_ranks}
        for r in my_ranks:
            a_host[r].copy_(comm.tensor(r, N.BUF_A_SHARD, prob).cpu())

        def e2e_step():
            for r in my_ranks:
                comm.copy_in(r, N.BUF_A_SHARD, prob, a_host[r].data_ptr(), a_host[r].shape[1], stream)
            op()
            for r in my_ranks:
                comm.copy_out(r, N.BUF_C_OUT, prob, c_host[r].data_ptr(), c_host[r].shape[1], stream)

        ms_serial = timed(e2e_step, max(3, args.steps // 2), 2)

        # Pipelined steps (the way a serving / training loop drives the op):
        # step i+1's A shards go host->device on one copy stream while step i
        # computes and step i-1's C goes device->host on another; caller-owned
        # double buffers through the public *_ex API. Every step still moves
        # its own inputs in and its result out inside the timed region.
        s_h2d, s_d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        cs = torch.cuda.current_stream()
        a_dev = [{r: torch.empty_like(a_host[r], device=dev) for r in my_ranks} for _ in range(2)]
        c_dev = [{r: torch.empty(c_host[r].shape, dtype=torch.bfloat16, device=dev) for r in my_ranks} for _ in range(2)]
        w_views = {r: comm.tensor(r, N.BUF_B_SHARD, prob) for r in my_ranks}
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]

        def op_ex(b):
            ops_list = [(a_dev[b][r], w_views[r], c_dev[b][r]) for r in my_ranks]
            if pattern == 0:
                comm.ag_gemm_ex(prob, tile, ops_list, prob.rows_per_rank(), fx.PULL, True, opts, streams)
            else:
                comm.gemm_rs_ex(prob, tile, ops_list, args.write_mode, True, opts, streams)

        def h2d(b):
            with torch.cuda.stream(s_h2d):
                for r in my_ranks:
                    a_dev[b][r].copy_(a_host[r], non_blocking=True)
                ev_in[b].record(s_h2d)

        def pipelined(steps):
            h2d(0)
            for i in range(steps):
                b = i % 2
                if i + 1 < steps:
                    if i >= 1:
                        s_h2d.wait_event(ev_done[1 - b])  # step i-1 no longer reads that buffer
                    h2d(1 - b)
                cs.wait_event(ev_in[b])
                if i >= 2:
                    cs.wait_event(ev_out[b])  # step i-2's result has left that buffer
                op_ex(b)
                ev_done[b].record(cs)
                s_d2h.wait_event(ev_done[b])
                with torch.cuda.stream(s_d2h):
                    for r in my_ranks:
                        c_host[r].copy_(c_dev[b][r], non_blocking=True)
                    ev_out[b].record(s_d2h)

        n_e2e = max(3, args.steps // 2)
        pipelined(2)  # warm-up
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(s_h2d)
        s_h2d.wait_event(t0)
        pipelined(n_e2e)
        t1.record(s_d2h)
        t1.synchronize()
        barrier()
        tt_ms = torch.tensor([t0.elapsed_time(t1) / n_e2e], device=dev)
        if dist is not None:
            dist.all_reduce(tt_ms, op=dist.ReduceOp.MAX)
        ms_e2e = tt_ms.item()
        h2d_b = sum(t.numel() * 2 for t in a_host.values())
        d2h_b = sum(t.numel() * 2 for t in c_host.values())
        if dist is not None:
            tt = torch.tensor([h2d_b, d2h_b], device=dev, dtype=torch.float64)
            dist.all_reduce(tt)
            h2d_b, d2h_b = int(tt[0].item()), int(tt[1].item())
        e2e = {"value": flops / (ms_e2e * 1e-3) / 1e12, "unit": "TFLOPS", "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b,
               "path": "pinned host A shards -> device (copy stream) | flux_ag_gemm_ex / flux_gemm_rs_ex on caller "
                       "buffers | C -> pinned host (second copy stream); steps pipelined, double-buffered",
               "serial_ms_per_step": ms_serial,
               "serial_path": "flux_copy_in -> fused op -> flux_copy_out, one stream, no overlap"}

    # ---- roofline of the dominant kernel (the fused GEMM) ----
    pk, src = peaks()
    kms = statistics.mean(kernel_ms) if kernel_ms else ms_fused
    roofline = roofline_of(roofline_work(pattern, m, n, k, tp, emulated), kms, pk, src)
    # Which kernel ran, by the library's auto rule (stream_kernel_ok, flux_api.cpp):
    # the streaming decode kernel for <= 128 GEMM rows with one rank per launch.
    per_launch = tp if emulated else 1
    if per_launch == 1 and m <= 128:
        roofline["kernel"] = "flux_stream_kernel<AG>" if pattern == 0 else "flux_stream_kernel<RS>"
    else:
        roofline["kernel"] = "flux_gemm_kernel<AG>" if pattern == 0 else "flux_gemm_kernel<RS>"
    roofline["traffic"] = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof) and emulated:  # captured at N=1 (every rank in one launch)
        try:
            with open(prof) as f:
                tr = json.load(f)
            roofline["traffic"] = tr.get(wl)
            if roofline["traffic"] is not None:
                roofline["traffic_source"] = tr.get("_source", "profiles/ncu_traffic.json (ncu --set full capture)")
        except Exception:
            roofline["traffic"] = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = run_cpu_reference(pattern, m, n, k, tp)
        except Exception as e:  # reported, never fatal for the GPU number
            cpu = {"value": None, "unit": "TFLOPS", "cores": 0, "kind": "unavailable", "sample": repr(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_fused, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform[-1,1) bf16)",
            "config": {"workload": wl, "description": desc, "m": m, "n": n, "k": k, "tp": tp,
                       "ranks": "emulated on one GPU" if emulated else "one process per GPU (cudaIpc heaps)",
                       "parallelism": f"tp{tp}",
                       "transfer": ("NVLS " + nvls_note if nvls_mode != fx.NVLS_OFF else
                                    (ag_transfer if pattern == 0 else "epilogue P2P")),
                       "l2": "flushed between timed steps outside the events (256 MiB write, then a 256 MiB read "
                             "sweep so no dirty lines drain inside the timed region)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "parity": parity,
            "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary(), "overlap": extra,
        }
        if args.nvls:
            line["nvls"] = nvls_note
        print(json.dumps(line), flush=True)
    comm.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="llama70b-up-ag")
    ap.add_argument("--quick", action="store_true", help="headline number only")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ag-engine", type=int, default=0, help="0 auto, 1 copy engines, 2 in-kernel (SM) transfers")
    ap.add_argument("--cta-group", type=int, default=0, help="0 auto, 1 single-CTA tiles, 2 CTA pairs")
    ap.add_argument("--write-mode", type=int, default=0, help="RS: 0 WriteAlltoAll, 1 FusedReduce")
    ap.add_argument("--nvls", type=int, default=0, help="1: NVLS multicast (emulated when ranks share one GPU)")
    ap.add_argument("--nondeterministic", action="store_true", help="RS FusedReduce in arrival order (red.add)")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args, args.workload)
    else:
        our_arm(args, args.workload)


if __name__ == "__main__":
    main()
