#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1800 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_default.err
timeout 900 python bench.py --gpus 2 --one-device --workload llama70b32k --steps 3 --warmup 3 --no-side --no-cpu-baseline \
  --no-hbm-tier --no-l1-reuse > gpurun_out/bench_2rank_onedev.json 2> gpurun_out/bench_2rank_onedev.err; echo "bench 2rank rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench ref rc=$?"
