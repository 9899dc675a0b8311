#!/bin/bash
# ncu evidence for the value arm's kernel + the bench launch list, and the K1 grid/U sweep:
#   gpurun --timeout 2400 -- 'bash tools/ncu_r01b.sh'
mkdir -p gpurun_out
for sh in qwen 8b 70b 70b_tp2 70b_tp8; do SHAPE=$sh python tools/k1_sweep.py 296 592 1184 2368 4736; done > gpurun_out/k1_sweep.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ingest_ldg -s 1 -c 1 -o gpurun_out/prof_k1hbm python tools/prof_targets.py ingest-hbm > gpurun_out/prof_k1hbm.log 2>&1; echo "ncu k1hbm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ingest_ldg -s 1 -c 1 -o gpurun_out/prof_k1hbm_tp8 python tools/prof_targets.py ingest-hbm-tp8 > gpurun_out/prof_k1hbm_tp8.log 2>&1; echo "ncu k1hbm tp8 rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_bench_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-alt-modes > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
