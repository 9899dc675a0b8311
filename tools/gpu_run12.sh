mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_prefix -c 1 -o gpurun_out/prof_hash2 python tools/prof_targets.py hash > /dev/null 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tile_sort|k_merge_pass" -c 2 -o gpurun_out/prof_sort python tools/prof_targets.py scorer > /dev/null 2>&1; echo "ncu rc=$?"
