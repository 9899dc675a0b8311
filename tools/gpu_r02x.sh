#!/bin/bash
# Round 2 (after the batched-memcpy calls were closed on the pool): CE probes with per-call
# copies, the GPU suite, smoke, the contract bench line, the reference arm.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ce_direct_probe tools/probe/ce_direct_probe.cu && timeout 300 /tmp/ce_direct_probe > gpurun_out/x_ce_percall_probe.jsonl 2>&1; echo "ce probe rc=$?"
timeout 300 python tools/probe/overlap_probe.py > gpurun_out/x_overlap_probe.jsonl 2>&1; echo "overlap rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/x_pytest_gpu.log 2>&1
echo "pytest -m gpu rc=$?"; tail -3 gpurun_out/x_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/x_bench.json 2> gpurun_out/x_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/x_bench_ref.json 2> gpurun_out/x_bench_ref.err; echo "bench ref rc=$?"
