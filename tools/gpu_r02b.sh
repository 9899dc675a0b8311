#!/bin/bash
# Round-2 second GPU pass: new tests (stage modes + L3, full-size parity, K7 determinism), the full
# GPU suite, and the default bench.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage_modes.py tests/test_gpu_fullsize.py tests/test_gpu_index.py -q -p no:cacheprovider > gpurun_out/pytest_new.log 2>&1
echo "pytest new rc=$?"; tail -30 gpurun_out/pytest_new.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest -m gpu rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_default.err
