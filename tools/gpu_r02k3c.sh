#!/bin/bash
# Round 2: K3 chain with CTA-local length ranking -- hash parity tests, then the configs[4] sweep.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "hash" > gpurun_out/k3c_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/k3c_pytest.log
timeout 600 python tools/k3_sweep.py > gpurun_out/k3c_sweep.jsonl 2> gpurun_out/k3c_sweep.err; echo "sweep rc=$?"; cat gpurun_out/k3c_sweep.jsonl
timeout 600 ncu --set full --clock-control none -k regex:k_chain -c 1 -f -o gpurun_out/k3c_prof_chain python tools/prof_targets.py hash > /dev/null 2>&1; echo "ncu rc=$?"
