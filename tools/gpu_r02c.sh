#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage_modes.py tests/test_gpu_consumer.py -q -p no:cacheprovider > gpurun_out/pytest_new.log 2>&1
echo "pytest new rc=$?"; tail -30 gpurun_out/pytest_new.log
timeout 1800 python tools/bench_mixed.py --consumer real --n 24 --profile gpurun_out/r02_mixed_real_timeline.json > gpurun_out/r02_mixed_real.json 2> gpurun_out/r02_mixed_real.err; echo "mixed real rc=$?"; tail -c 1200 gpurun_out/r02_mixed_real.err
timeout 1200 python tools/bench_calibrate.py > gpurun_out/r02_calibrate.json 2> gpurun_out/r02_calibrate.err; echo "calibrate rc=$?"; tail -c 1200 gpurun_out/r02_calibrate.err
