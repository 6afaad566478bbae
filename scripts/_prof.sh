FLUX_SERIALIZE_TRANSFERS=1 ncu --set full --clock-control none --import-source on -k regex:flux_gemm_kernel -s 1 -c 1 -o gpurun_out/ag_llama70b_up_tp8 python scripts/profile_op.py --workload llama70b-up-ag --iters 2 > gpurun_out/ncu_ag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:flux_gemm_kernel -s 1 -c 1 -o gpurun_out/rs_llama70b_down_tp8 python scripts/profile_op.py --workload llama70b-down-rs --iters 2 > gpurun_out/ncu_rs.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:flux_gemm_kernel -s 1 -c 1 -o gpurun_out/local_gemm_llama70b_up_tp8 python scripts/profile_op.py --workload llama70b-up-ag --op local --iters 2 > gpurun_out/ncu_local.log 2>&1
FLUX_SERIALIZE_TRANSFERS=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_ag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --quick > gpurun_out/ncu_launch_ag.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_rs.csv python bench.py --workload llama70b-down-rs --steps 2 --warmup 3 --no-cpu-baseline --quick > gpurun_out/ncu_launch_rs.log 2>&1
ls gpurun_out
