set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python tools/microbench.py > gpurun_out/microbench2.log 2>&1; echo "mb rc=$?"; cat gpurun_out/microbench2.log | grep "^{"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_scorer_launches.csv python tools/prof_targets.py scorer > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_prefix -c 1 -o gpurun_out/prof_hash python tools/prof_targets.py hash > /dev/null 2>&1; echo "ncu2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ingest_ldg -s 8 -c 1 -o gpurun_out/prof_k2 python tools/prof_targets.py ingest-ce > /dev/null 2>&1; echo "ncu3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ingest_bulk -s 4 -c 1 -o gpurun_out/prof_bulk python tools/prof_targets.py ingest-bulk > /dev/null 2>&1; echo "ncu4 rc=$?"
ls -la gpurun_out
