timeout 600 python -m pytest tests/test_stream_gpu.py tests/test_nvls_gpu.py -x -q 2>&1 | tail -3
for cl in 1 0 2 4; do
for args in "0 16 3584 8192 1" "1 16 8192 3584 1" "1 16 8192 1024 1" "1 64 8192 3584 1"; do
  echo "== cl=$cl $args"
  FLUX_SK_CLUSTER=$cl timeout 120 python scripts/stream_trace.py $args 2>&1 | grep -E "kernel|cta end|Error|error" | tail -3
done; done
