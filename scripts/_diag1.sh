timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for args in "1 16 8192 1024 1" "1 16 8192 3584 1" "0 16 3584 8192 1" "1 1024 1024 1024 2"; do
  echo "== $args"
  timeout 120 python scripts/stream_trace.py $args 2>&1 | grep -v "warp [4567]"
done
