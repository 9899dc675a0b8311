#!/bin/bash
# ncu --set full captures of every kernel family on the final code (one GPU, short targets):
#   gpurun --timeout 2400 -- 'bash tools/ncu_full.sh'   then   python tools/ncu_summarize.py
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:"k_chunk_digest|k_chain" -c 2 -o gpurun_out/prof_hash -f python tools/prof_targets.py hash > /dev/null 2>&1; echo "hash rc=$?"
timeout 900 $N -k regex:"k_score|k_check_sorted|k_tile_sort|k_merge_pass|k_iota" -c 6 -o gpurun_out/prof_score -f python tools/prof_targets.py scorer > /dev/null 2>&1; echo "score rc=$?"
timeout 900 $N -k regex:k_ingest_ldg -s 2 -c 1 -o gpurun_out/prof_k2 -f python tools/prof_targets.py ingest-ce > /dev/null 2>&1; echo "k2 rc=$?"
timeout 900 $N -k regex:k_ingest_bulk -c 1 -o gpurun_out/prof_bulk -f python tools/prof_targets.py ingest-bulk > /dev/null 2>&1; echo "bulk rc=$?"
timeout 900 $N -k regex:k_ingest_ldg -s 1 -c 1 -o gpurun_out/prof_k1hbm -f python tools/prof_targets.py ingest-hbm > /dev/null 2>&1; echo "k1hbm rc=$?"
timeout 900 $N -k regex:"k_index" -c 2 -o gpurun_out/prof_index -f python tools/prof_targets.py index > /dev/null 2>&1; echo "index rc=$?"
