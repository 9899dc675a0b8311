#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python bench.py --workload llama8b32k --steps 3 --warmup 2 --no-side --no-cpu-baseline --no-hbm-tier > gpurun_out/bench_8b.json 2> gpurun_out/bench_8b.err; echo "bench 8b rc=$?"; tail -c 400 gpurun_out/bench_8b.err
python -c "import json; d=json.loads(open('gpurun_out/bench_8b.json').read().strip().splitlines()[-1]); print(d['value'], json.dumps(d['l1_reuse']))"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest -m gpu rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
