#!/bin/bash
# Round-2 measurement batch (one gpurun call): bench lines for the headline and
# the decode / C1 workloads, the ncu launch list of the headline command, and
# ncu --set full captures of the fused AG kernel with the in-kernel transfer
# live and of the streaming decode kernel (GEMM-RS, one GPU's share).
set -x
O=gpurun_out/r2
mkdir -p $O
timeout 600 python bench.py > $O/bench_llama70b-up-ag.json 2> $O/bench_headline.err
for wl in rank-decode-ag-up-m16 rank-decode-rs-down-m16 rank-decode-rs-attn-m16 decode-ag-up-m16 decode-rs-down-m16 rs-1024-tp2 llama70b-down-rs; do
  timeout 300 python bench.py --workload $wl --no-cpu-baseline > $O/bench_$wl.json 2> $O/bench_$wl.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_headline.csv python bench.py --steps 2 --warmup 1 --quick --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:flux_gemm_kernel -s 2 -c 1 -o $O/ag_llama70b_up_tp8_smengine python bench.py --steps 1 --warmup 2 --quick --no-cpu-baseline --ag-engine 2 > $O/ncu_ag.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:flux_stream_kernel -s 2 -c 1 -o $O/stream_rank_rs_down_m16 python bench.py --steps 1 --warmup 2 --quick --no-cpu-baseline --workload rank-decode-rs-down-m16 > $O/ncu_stream.log 2>&1
ls -la $O
