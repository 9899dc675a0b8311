#!/bin/bash
# Round 2: A/B on one box -- the stage under a prefill with CE + K2 (AUTO) vs per-call CE-direct,
# real consumer and K6.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for rep in 1 2; do
for m in auto ce_direct; do
  timeout 900 python tools/bench_mixed.py --consumer real --n 24 --mode $m > gpurun_out/z_mixed_real_${m}_${rep}.json 2> gpurun_out/z_mixed_real_${m}_${rep}.err; echo "real $m $rep rc=$?"
  timeout 900 python tools/bench_mixed.py --compute-per-token 4e-6 --mode $m > gpurun_out/z_mixed_k6_${m}_${rep}.json 2> gpurun_out/z_mixed_k6_${m}_${rep}.err; echo "k6 $m $rep rc=$?"
done
done
