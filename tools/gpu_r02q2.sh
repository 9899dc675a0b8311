#!/bin/bash
# Round 2: why does K6 start later beside CE + K2?  Hypothesis: K2 launches waiting (in-stream)
# on a long CE copy block a hardware queue the compute stream shares.  Vary the staging ring
# (shorter waits) and CUDA_DEVICE_MAX_CONNECTIONS (more hardware queues).
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for st in 1024 256 64; do
  timeout 900 python tools/bench_mixed.py --compute-per-token 4e-6 --staging-mib $st > gpurun_out/q2_k6_st${st}.json 2> gpurun_out/q2_k6_st${st}.err; echo "k6 staging $st rc=$?"
done
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 900 python tools/bench_mixed.py --compute-per-token 4e-6 > gpurun_out/q2_k6_conn32.json 2> gpurun_out/q2_k6_conn32.err; echo "k6 conn32 rc=$?"
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 900 python tools/bench_mixed.py --compute-per-token 4e-6 --mode ce_direct > gpurun_out/q2_k6_conn32_cedirect.json 2> gpurun_out/q2_k6_conn32_cedirect.err; echo "k6 conn32 ce_direct rc=$?"
timeout 900 python tools/bench_mixed.py --consumer real --n 24 --staging-mib 64 > gpurun_out/q2_real_st64.json 2> gpurun_out/q2_real_st64.err; echo "real staging 64 rc=$?"
