#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 300 tools/probe/ce_direct_probe 4096 > gpurun_out/r02_ce_direct_probe.jsonl 2>&1; echo "ce direct rc=$?"; cat gpurun_out/r02_ce_direct_probe.jsonl
timeout 900 python tools/bench_peer.py > gpurun_out/r02_peer_tier.jsonl 2> gpurun_out/r02_peer_tier.err; echo "peer rc=$?"; cut -c1-200 gpurun_out/r02_peer_tier.jsonl
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest -m gpu rc=$?"; tail -5 gpurun_out/pytest_gpu.log
