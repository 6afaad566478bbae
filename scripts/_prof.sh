timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
timeout 600 python scripts/decode_sweep.py --iters 20 --out gpurun_out/decode_sweep.json > gpurun_out/dec.log 2>&1; tail -1 gpurun_out/dec.log
ncu --set full --clock-control none --import-source on -k regex:flux_gemm_kernel -s 1 -c 1 -o gpurun_out/rs_llama70b_down_tp8 python scripts/profile_op.py --workload llama70b-down-rs --iters 2 > gpurun_out/ncu_rs.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_rs_r1b.csv python bench.py --workload llama70b-down-rs --steps 2 --warmup 3 --no-cpu-baseline --quick > gpurun_out/ncu_launch_rs.log 2>&1
ls gpurun_out
