#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 300 tools/probe/ce_direct_probe 4096 > gpurun_out/r02_ce_direct_probe.jsonl 2>&1; echo "ce direct rc=$?"; cat gpurun_out/r02_ce_direct_probe.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stage_modes.py tests/test_gpu_consumer.py tests/test_gpu_stage_random.py tests/test_gpu_peer.py tests/test_cpp_api.py -q -x -p no:cacheprovider > gpurun_out/pytest_new.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_new.log
timeout 900 python tools/bench_peer.py > gpurun_out/r02_peer_tier.jsonl 2> gpurun_out/r02_peer_tier.err; echo "peer rc=$?"; cat gpurun_out/r02_peer_tier.jsonl | cut -c1-260
timeout 1800 python tools/bench_mixed.py --consumer real --n 24 --profile gpurun_out/r02_mixed_real_timeline.json > gpurun_out/r02_mixed_real.json 2> gpurun_out/r02_mixed_real.err; echo "mixed real rc=$?"; tail -c 600 gpurun_out/r02_mixed_real.err
timeout 1200 python tools/bench_calibrate.py > gpurun_out/r02_calibrate.json 2> gpurun_out/r02_calibrate.err; echo "calibrate rc=$?"; tail -c 600 gpurun_out/r02_calibrate.err
