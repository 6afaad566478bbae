O=gpurun_out/r2; mkdir -p $O
FLUX_SERIALIZE_TRANSFERS=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_headline_serialized.csv python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline > $O/launch_ser.out 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_headline_smengine.csv python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline --ag-engine 2 > $O/launch_sm.out 2>&1
tail -c 300 $O/launch_ser.out; tail -c 300 $O/launch_sm.out
