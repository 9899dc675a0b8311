#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_stage_modes.py tests/test_gpu_consumer.py -q -p no:cacheprovider -x > gpurun_out/pytest_stage.log 2>&1
echo "pytest stage rc=$?"; tail -3 gpurun_out/pytest_stage.log
timeout 1800 python tools/bench_mixed.py --consumer real --n 24 --profile gpurun_out/r02_mixed_real_timeline.json > gpurun_out/r02_mixed_real.json 2> gpurun_out/r02_mixed_real.err; echo "mixed real rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_mixed_real.json')); print(json.dumps(d['runs'])); print(d.get('sim_vs_real'))"
timeout 900 python tools/bench_mixed.py --compute-per-token 4e-6 > gpurun_out/r02_mixed_k6.json 2> /dev/null; echo "mixed k6 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_mixed_k6.json')); print(json.dumps(d['runs'])); print(d.get('sim_vs_real'))"
