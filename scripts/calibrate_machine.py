"""Calibrate the reference simulator's MachineModel on this B200 (SPEC.md:304,
SURVEY.md §8f row 4) and write it in the reference's config schema.

* compute: our plain local GEMM (tp=1) at K=8192 for 1..6 full waves of
  128x256 tiles over the 148 SMs -> per-slot flops_per_us (wave model fit);
* launch_overhead_us: the smallest possible operator (one 128x256x64 tile);
* link: single copy-engine transfers (cudaMemcpyAsync device-to-device) of
  1..256 MiB -> latency + bandwidth. With one GPU this is the emulated link
  (HBM read+write), not NVLink 5; the file says so;
* split efficiency: the L-AG local GEMM (M=4096, N=3584, K=8192) whole vs one
  M/P row chunk, P = 2, 4, 8 (simulate_medium's chunk model).

    python scripts/calibrate_machine.py --out profiles/round1/machine_b200.json
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from cuda.bindings import runtime as cudart

import paper_2406_06858_b200 as fx
from paper_2406_06858_b200 import _native as N
from paper_2406_06858_b200 import calibrate as CAL

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="")
ap.add_argument("--iters", type=int, default=20)
args = ap.parse_args()
torch.cuda.set_stream(torch.cuda.Stream())
stream = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
SMS = torch.cuda.get_device_properties(0).multi_processor_count


def timed_us(fn, iters=args.iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.zero_()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def local_gemm_us(m, n, k):
    p = fx.ProblemSpec(m, n, k, 1, fx.ALLGATHER_GEMM)
    comm = fx.Communicator(1, [0], heap_bytes=fx.required_heap_bytes(p) + (16 << 20))
    for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
        t = comm.tensor(0, kind, p)
        t.copy_(torch.rand(t.shape, device="cuda").mul_(2).sub_(1))
    st = [stream.cuda_stream]
    us = timed_us(lambda: comm.local_gemm(p, None, st))
    comm.sync()
    comm.close()
    return us


TM, TN, K = 128, 256, 8192
n_cols = TN * (SMS // 4)  # 37 column tiles: 4 tile rows per wave
compute = []
for waves in (1, 2, 3, 4, 6):
    m = TM * 4 * waves
    tiles = (m // TM) * (n_cols // TN)
    compute.append((tiles, local_gemm_us(m, n_cols, K)))
    print("compute", m, n_cols, K, tiles, compute[-1][1], flush=True)
intercept, flops_per_us = CAL.fit_compute(compute, SMS, TM, TN, K)
launch_us = local_gemm_us(128, 256, 64)
print("launch", launch_us, "intercept", intercept, flush=True)

link = []
for mib in (1, 4, 16, 64, 256):
    nbytes = mib << 20
    src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src)

    def copy():
        err, = cudart.cudaMemcpyAsync(dst.data_ptr(), src.data_ptr(), nbytes,
                                      cudart.cudaMemcpyKind.cudaMemcpyDeviceToDevice, stream.cuda_stream)
        assert err == cudart.cudaError_t.cudaSuccess, err
    link.append((nbytes, timed_us(copy)))
    print("link", nbytes, link[-1][1], flush=True)
    del src, dst
link_lat, link_bw = CAL.fit_link(link)

t_full = local_gemm_us(4096, 3584, K)
chunks = {p: local_gemm_us(4096 // p, 3584, K) for p in (2, 4, 8)}
split = CAL.fit_split_efficiency(CAL.split_efficiency_samples(t_full, chunks))
print("split", t_full, chunks, split, flush=True)

machine = CAL.MachineModel(sm_count=SMS, flops_per_us=flops_per_us, launch_overhead_us=launch_us,
                           link_bw_bytes_per_us=link_bw, link_latency_us=link_lat, bytes_per_element=2,
                           split_efficiency=split)
cfg = CAL.reference_config(
    machine, {"m": 4096, "n": 28672, "k": 8192, "tp": 8, "pattern": "AllGatherGemm"}, {"tm": TM, "tn": TN},
    {"gpu": torch.cuda.get_device_name(0), "sms": SMS,
     "compute_samples_tiles_us": compute, "compute_fit_intercept_us": intercept,
     "launch_probe": "one 128x256x64 tile, median of %d, L2 flushed" % args.iters,
     "link_samples_bytes_us": link,
     "link_note": "copy-engine device-to-device on ONE B200 (the emulated link: HBM read + write); "
                  "NVLink 5 is 900 GB/s per direction = 9e5 bytes/us",
     "split_samples": {"t_full_us": t_full, "chunk_us_by_partitions": chunks},
     "gemm": "flux_local_gemm (tcgen05, this repo), bf16 in, fp32 accumulate"})
print(json.dumps(cfg["config"]["machine"], indent=1))
if args.out:
    json.dump(cfg, open(args.out, "w"), indent=1)
