#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "hash" 2>&1 | tail -4
timeout 600 python tools/k3_sweep.py > gpurun_out/r02_k3_chain.jsonl 2> gpurun_out/k3.err; echo "k3 rc=$?"; tail -3 gpurun_out/k3.err
cat gpurun_out/r02_k3_chain.jsonl
