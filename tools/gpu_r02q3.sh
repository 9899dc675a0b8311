#!/bin/bash
# Round 2: CE staging-group size under a prefill (K6 and the real consumer), two reps.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for rep in 1 2; do
for st in 1024 512 256 128; do
  timeout 900 python tools/bench_mixed.py --compute-per-token 4e-6 --staging-mib $st > gpurun_out/q3_k6_st${st}_${rep}.json 2> /dev/null; echo "k6 $st $rep rc=$?"
  timeout 900 python tools/bench_mixed.py --consumer real --n 24 --staging-mib $st > gpurun_out/q3_real_st${st}_${rep}.json 2> /dev/null; echo "real $st $rep rc=$?"
done
done
