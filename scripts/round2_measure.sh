#!/bin/bash
# Round-2 measurement batch (one gpurun call): smoke, bench lines for the
# headline and the decode / C1 workloads, and the decode sweep.
set -x
O=gpurun_out/r2f
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_llama70b-up-ag.json 2> $O/bench_headline.err
for wl in rank-decode-ag-up-m16 rank-decode-rs-down-m16 rank-decode-rs-attn-m16 rank-decode-ag-up-m128 decode-ag-up-m16 decode-rs-down-m16 rs-1024-tp2 llama70b-down-rs; do
  timeout 300 python bench.py --workload $wl --no-cpu-baseline > $O/bench_$wl.json 2> $O/bench_$wl.err
done
timeout 900 python scripts/decode_sweep.py --out $O/decode_sweep.json > $O/decode_sweep.log 2>&1
ls -la $O
