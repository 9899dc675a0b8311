set -x
mkdir -p gpurun_out
# launch list of the bench command (cold, serialised -- shares only)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_bench_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.json 2>/dev/null; echo "ncu-launch rc=$?"
# full set on the dominant kernel (K2) inside the bench
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_ingest_ldg -s 200 -c 1 -o gpurun_out/prof_bench_k2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --workload llama8b32k > /dev/null 2>&1; echo "ncu-full rc=$?"
ls -la gpurun_out
