#!/bin/bash
# Round 2: layer pipelining with the real consumer (attention pre-planned, page lists filled from
# the device block table): uniform batches where one request's ingest and prefill are comparable,
# and the configs[3] mixed trace; serial vs per-layer-fenced prefill.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_consumer.py tests/test_gpu_stage.py -q -p no:cacheprovider -x > gpurun_out/lp4_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/lp4_pytest.log
for spec in 12:32768:0.97 12:32768:0.98 8:65536:0.985 12:32768:0.9; do
  n=${spec%%:*}; u=${spec#*:}
  tag=$(echo $spec | tr ':.' '__')
  timeout 900 python tools/bench_mixed.py --consumer real --n $n --uniform $u > gpurun_out/lp4_real_${tag}.json 2> gpurun_out/lp4_real_${tag}.err; echo "real $spec rc=$?"
done
timeout 1800 python tools/bench_mixed.py --consumer real --n 24 --profile gpurun_out/lp4_mixed_real_timeline.json > gpurun_out/lp4_mixed_real.json 2> gpurun_out/lp4_mixed_real.err; echo "mixed real rc=$?"
