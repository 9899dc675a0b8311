#!/bin/bash
# Round 2: the stage's CE group cap under a prefill -- tests, configs[3] (K6 and real consumer),
# CALVO comparison, on the final stage code.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_stage_modes.py tests/test_gpu_stage_random.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/w2_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/w2_pytest.log
timeout 900 python tools/bench_mixed.py --compute-per-token 4e-6 > gpurun_out/w2_mixed_k6.json 2> /dev/null; echo "k6 rc=$?"
timeout 1800 python tools/bench_mixed.py --consumer real --n 24 --profile gpurun_out/w2_mixed_real_timeline.json > gpurun_out/w2_mixed_real.json 2> /dev/null; echo "real rc=$?"
timeout 1500 python tools/bench_calvo.py > gpurun_out/w2_calvo.json 2> gpurun_out/w2_calvo.err; echo "calvo rc=$?"
