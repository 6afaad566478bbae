timeout 600 python -m pytest tests/test_stream_gpu.py tests/test_nvls_gpu.py -x -q 2>&1 | tail -2
for rep in 1 2; do
for dbg in 0 1024; do
for args in "1 16 8192 3584 1" "1 16 8192 1024 1" "1 16 8192 3584 8"; do
  echo "== dbg=$dbg $args"
  FLUX_DEBUG=$dbg timeout 120 python scripts/stream_trace.py $args 2>&1 | grep -E "kernel" | tail -2
done; done; done
