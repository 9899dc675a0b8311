#!/bin/bash
# compute-sanitizer over the round-2 kernels and stage paths: K1b tensor-map TMA (NHD/HND, host and
# HBM sources, as K2), CE-direct, K8 replication, the destination-side page check, the K7
# deterministic insert / compaction, the hash phases, and the stage with L3 + modes.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
SEL="k1b or ce_direct or hash_aligned or layouts"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --kernel-name-exclude kns=at::,kns=void_at,kns=elementwise,kns=vectorized \
    python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "$SEL" > gpurun_out/r02_sanitize_$tool.log 2>&1
  echo "$tool parity rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r02_sanitize_$tool.log | tail -2
done
timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 --kernel-name-exclude kns=at::,kns=void_at,kns=elementwise,kns=vectorized \
  python -m pytest tests/test_gpu_stage.py tests/test_gpu_stage_modes.py tests/test_gpu_index.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x \
  -k "not decoupled_beats_coupled" > gpurun_out/r02_sanitize_memcheck_stage.log 2>&1
echo "memcheck stage rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r02_sanitize_memcheck_stage.log | tail -2
