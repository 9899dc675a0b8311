mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ingest_ldg -s 1 -c 1 -o gpurun_out/prof_k1hbm python tools/prof_targets.py ingest-hbm > gpurun_out/prof_k1hbm.log 2>&1; echo "ncu k1hbm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ingest_ldg -s 1 -c 1 -o gpurun_out/prof_k1hbm_tp8 python tools/prof_targets.py ingest-hbm-tp8 > gpurun_out/prof_k1hbm_tp8.log 2>&1; echo "ncu k1hbm tp8 rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_bench_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-alt-modes > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
