set -x
mkdir -p gpurun_out
timeout 600 python tools/k2_sweep.py 2>&1 | grep "^{"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_ingest_ldg -s 40 -c 1 -o gpurun_out/prof_bench_k2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --workload llama8b32k > /dev/null 2>&1; echo "ncu-full rc=$?"
ls gpurun_out
