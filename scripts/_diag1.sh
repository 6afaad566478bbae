timeout 600 python -m pytest tests/test_stream_gpu.py -x -q 2>&1 | tail -2
for args in "1 64 8192 3584 1" "1 16 8192 3584 1" "1 16 8192 1024 1"; do
  echo "== $args"
  timeout 120 python scripts/stream_trace.py $args 2>&1 | grep -E "kernel" | tail -2
done
