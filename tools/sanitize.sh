mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --kernel-name-exclude kns=at::,kns=void_at,kns=elementwise,kns=vectorized python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x \
    -k "ingest_bit_exact or head_sharded or k2_scatter or hash_frozen or hash_random or hash_edge or scores_and_order or (large_queue_matches_oracle and 4097) or presorted or layouts or sparse_layer" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_$tool.log | tail -3
done
