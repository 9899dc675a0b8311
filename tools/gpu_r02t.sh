#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "hash" 2>&1 | tail -2 | tee gpurun_out/k3_tests.txt
timeout 600 python tools/k3_sweep.py > gpurun_out/r02_k3_fused.jsonl 2> gpurun_out/k3.err; echo "k3 rc=$?"; tail -3 gpurun_out/k3.err
python -c "
import json
for l in open('gpurun_out/r02_k3_fused.jsonl'):
    d=json.loads(l); print(d['layout'], d['ctas_per_sm'], d['prefetch_groups'], d['fused_chain'], round(d['phase1_ms'],3), round(d['total_ms'],3), round(d['total_read_ceiling_frac'],3))"
timeout 600 ncu --set full --clock-control none -k regex:"k_chunk_hash_fused|k_chain_tail" -s 2 -c 2 -o gpurun_out/k3_fused -f python tools/prof_k3.py 1 1 > gpurun_out/ncu_k3.log 2>&1; echo "ncu rc=$?"
