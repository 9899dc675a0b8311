#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 python tools/probe/overlap_probe.py > gpurun_out/r02_overlap_probe.jsonl 2> gpurun_out/r02_overlap_probe.err; echo "overlap rc=$?"; cat gpurun_out/r02_overlap_probe.jsonl; tail -c 600 gpurun_out/r02_overlap_probe.err
timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "reuse or copy_chunks or hash_aligned" > gpurun_out/pytest_new.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_new.log
timeout 1800 python tools/bench_mixed.py --consumer real --n 24 > gpurun_out/r02_mixed_real.json 2> gpurun_out/r02_mixed_real.err; echo "mixed real rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02_mixed_real.json')); print(json.dumps(d['runs']))"
