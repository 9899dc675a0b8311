#!/bin/bash
# Round 2: the stage keeps CE + K2 under a prefill (CE-direct by explicit mode only); refresh the
# stage tests, configs[3] with the real consumer (+ kineto timeline), the K6 mixed trace and the
# CALVO comparison on the new path.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_stage_random.py tests/test_gpu_stage.py tests/test_gpu_stage_modes.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/y_pytest_stage.log 2>&1
echo "pytest stage rc=$?"; tail -2 gpurun_out/y_pytest_stage.log
timeout 1800 python tools/bench_mixed.py --consumer real --n 24 --profile gpurun_out/y_mixed_real_timeline.json > gpurun_out/y_mixed_real.json 2> gpurun_out/y_mixed_real.err; echo "mixed real rc=$?"; tail -c 600 gpurun_out/y_mixed_real.err
timeout 900 python tools/bench_mixed.py --compute-per-token 4e-6 > gpurun_out/y_mixed_k6.json 2> gpurun_out/y_mixed_k6.err; echo "mixed k6 rc=$?"
timeout 1500 python tools/bench_calvo.py > gpurun_out/y_calvo.json 2> gpurun_out/y_calvo.err; echo "calvo rc=$?"; tail -c 600 gpurun_out/y_calvo.err
