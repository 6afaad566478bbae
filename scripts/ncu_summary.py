"""Summarise an ncu --set full capture into a small JSON (for profiles/)."""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__cluster_dim_x", "sm__cycles_elapsed.avg.per_second",
    "dram__cycles_elapsed.avg.per_second", "launch__shared_mem_per_block_dynamic",
]


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            out[k] = {"value": vals[i], "unit": units[i]}
    # top warp stall reasons (per-instruction-issued ratios)
    stalls = []
    for i, h in enumerate(hdr):
        pre = "smsp__average_warps_issue_stalled_"
        if h.startswith(pre) and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(vals[i]), h[len(pre):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    out["top_stalls"] = [{"reason": r, "ratio": v} for v, r in sorted(stalls, reverse=True)[:6]]
    return out


if __name__ == "__main__":
    res = {p: summarise(p) for p in sys.argv[1:]}
    print(json.dumps(res, indent=1))
