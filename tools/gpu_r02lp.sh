#!/bin/bash
# Round 2: layer pipelining with the real consumer where one request's ingest and prefill are
# comparable (uniform batches), serial vs per-layer-fenced prefill.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for u in 32768:0.9 65536:0.95 131072:0.98 16384:0.8; do
  tag=$(echo $u | tr ':.' '__')
  timeout 900 python tools/bench_mixed.py --consumer real --n 12 --uniform $u > gpurun_out/lp_real_${tag}.json 2> gpurun_out/lp_real_${tag}.err; echo "real $u rc=$?"
done
