#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest -m gpu rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 1800 python tools/bench_mixed.py --consumer real --n 24 --profile gpurun_out/r02_mixed_real_timeline.json > gpurun_out/r02_mixed_real.json 2> gpurun_out/r02_mixed_real.err; echo "mixed real rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_mixed_real.json')); print(json.dumps(d['runs'])); print(d['timeline'])"
timeout 900 python tools/bench_mixed.py --compute-per-token 4e-6 > gpurun_out/r02_mixed_k6.json 2> /dev/null; echo "mixed k6 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_mixed_k6.json')); print(json.dumps(d['runs'])); print(d.get('sim_vs_real'))"
