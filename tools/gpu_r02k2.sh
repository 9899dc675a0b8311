#!/bin/bash
# Round 2: K2 grid under a prefill (CE + K2 stage path): does a smaller scatter grid leave the
# prefill more SM room without slowing ingest?
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for c in 4736 1184 296 148 74; do
  timeout 900 python tools/bench_mixed.py --compute-per-token 4e-6 --k2-ctas $c > gpurun_out/k2g_mixed_k6_${c}.json 2> gpurun_out/k2g_mixed_k6_${c}.err; echo "k6 $c rc=$?"
  timeout 900 python tools/bench_mixed.py --consumer real --n 24 --k2-ctas $c > gpurun_out/k2g_mixed_real_${c}.json 2> gpurun_out/k2g_mixed_real_${c}.err; echo "real $c rc=$?"
done
