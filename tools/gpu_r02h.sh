#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_consumer.py -q -p no:cacheprovider > gpurun_out/pytest_stage.log 2>&1
echo "pytest stage rc=$?"; tail -15 gpurun_out/pytest_stage.log
timeout 1800 python tools/bench_mixed.py --consumer real --n 24 --profile gpurun_out/r02_mixed_real_timeline.json > gpurun_out/r02_mixed_real.json 2> gpurun_out/r02_mixed_real.err; echo "mixed real rc=$?"
timeout 1500 python bench.py --steps 5 --warmup 3 --no-side > gpurun_out/bench_reuse.json 2> gpurun_out/bench_reuse.err; echo "bench rc=$?"; tail -c 800 gpurun_out/bench_reuse.err
