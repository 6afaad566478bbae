"""Runs bench.py over every BASELINE.json config (ranks emulated on one GPU)
plus the decode sweep, and writes profiles/<round>/results.json + results.md."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
round_dir = sys.argv[1] if len(sys.argv) > 1 else "profiles/round1"
os.makedirs(os.path.join(ROOT, round_dir), exist_ok=True)
rows = []
for wl in ["llama70b-up-ag", "llama70b-down-rs", "llama70b-down-rs-tp4", "llama70b-down-rs-tp2", "gpt3-ag", "gpt3-rs",
           "rs-1024-tp2"]:
    out = subprocess.run([sys.executable, "bench.py", "--steps", "10", "--warmup", "3", "--no-cpu-baseline",
                          "--workload", wl], capture_output=True, text=True, cwd=ROOT, timeout=900)
    line = [l for l in out.stdout.splitlines() if l.startswith("{")]
    if not line:
        print(wl, "FAILED", out.stderr[-2000:])
        continue
    d = json.loads(line[-1])
    rows.append(d)
    print(wl, round(d["value"], 1), "TFLOPS", round(d["ms_per_step"], 3), "ms", flush=True)
json.dump(rows, open(os.path.join(ROOT, round_dir, "results.json"), "w"), indent=1)
md = ["| workload | TP | fused op (ms) | TFLOPS | kernel frac of peak | T_gemm ours / cuBLAS (ms) | B1 unfused (ms) | speedup vs B1 | Eq.2 overlap E | e2e TFLOPS |",
      "|---|---|---|---|---|---|---|---|---|---|"]
for d in rows:
    o = d.get("overlap", {})
    md.append(f"| {d['config']['workload']} | {d['config']['tp']} | {d['ms_per_step']:.3f} | {d['value']:.0f} | "
              f"{d['roofline']['frac']:.3f} | {o.get('t_gemm_ours_ms', 0):.3f} / {o.get('t_gemm_cublas_ms', 0):.3f} | "
              f"{o.get('t_unfused_cublas_ms', 0):.3f} | {o.get('speedup_vs_unfused', 0):.2f}x | "
              f"{o.get('overlap_efficiency', 0):.2f} | {d['e2e']['value']:.0f} |")
open(os.path.join(ROOT, round_dir, "results.md"), "w").write("\n".join(md) + "\n")
print("\n".join(md))
