#!/bin/bash
# Round-2 ncu evidence (one GPU): the launch list of the bench command and `--set full` captures
# of the kernels the round-2 numbers rest on.  Summaries: python tools/ncu_summarize_r02.py
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_ncu_bench_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-side --no-hbm-tier --no-alt-modes > /dev/null 2>&1; echo "launch list rc=$?"
N="ncu --set full --clock-control none --import-source on -f"
timeout 900 $N -k regex:k_ingest_ldg -s 2 -c 1 -o gpurun_out/r02_prof_k2 python tools/prof_targets.py ingest-ce > /dev/null 2>&1; echo "k2 rc=$?"
timeout 900 $N -k regex:k_ingest_tma -c 1 -o gpurun_out/r02_prof_k1b_tp8 python tools/prof_targets.py bulk-hbm-tp8 > /dev/null 2>&1; echo "k1b tp8 rc=$?"
timeout 900 $N -k regex:k_ingest_tma -c 1 -o gpurun_out/r02_prof_k1b_tp8_hnd python tools/prof_targets.py bulk-hbm-tp8-hnd > /dev/null 2>&1; echo "k1b tp8 hnd rc=$?"
timeout 900 $N -k regex:k_ingest_tma -c 1 -o gpurun_out/r02_prof_k1b_full python tools/prof_targets.py bulk-hbm > /dev/null 2>&1; echo "k1b full rc=$?"
timeout 900 $N -k regex:"k_chunk_digest|k_chain" -c 2 -o gpurun_out/r02_prof_hash python tools/prof_targets.py hash > /dev/null 2>&1; echo "hash rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_ncu_ce_direct_launches.csv \
  python tools/prof_targets.py ingest-ce-direct > /dev/null 2>&1; echo "ce direct launch list rc=$?"
