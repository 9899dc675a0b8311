#!/bin/bash
# Round 2: layer pipelining with the real consumer where one request's ingest and prefill are
# comparable (uniform batches), serial vs per-layer-fenced prefill.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for spec in 12:32768:0.97 12:32768:0.98 8:65536:0.985 12:32768:0.9 8:131072:0.98; do
  n=${spec%%:*}; u=${spec#*:}
  tag=$(echo $spec | tr ':.' '__')
  timeout 900 python tools/bench_mixed.py --consumer real --n $n --uniform $u > gpurun_out/lp2_real_${tag}.json 2> gpurun_out/lp2_real_${tag}.err; echo "real $spec rc=$?"
done
