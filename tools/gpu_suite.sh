#!/bin/bash
# One-GPU validation + measurement suite, run on a B200 box via gpurun:
#   gpurun --timeout 3000 -- 'bash tools/gpu_suite.sh [tests] [bench] [tools] [ncu]'
# Outputs land in gpurun_out/ (copy what should be judged into profiles/).
set -u
mkdir -p gpurun_out
steps="${*:-tests bench tools ncu}"
for s in $steps; do
  case $s in
    tests)
      timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
      echo "pytest -m gpu rc=$?"; tail -3 gpurun_out/pytest_gpu.log
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 ;;
    bench)
      timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
      timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> /dev/null; echo "bench ref rc=$?"
      timeout 600 python bench.py --workload llama8b32k > gpurun_out/bench_llama8b.json 2> /dev/null; echo "bench 8b rc=$?"
      timeout 900 python bench.py --workload llama70b32k > gpurun_out/bench_70b.json 2> /dev/null; echo "bench 70b rc=$?"
      timeout 900 python bench.py --hbm-tier-chunks 46 --no-cpu-baseline --no-alt-modes > gpurun_out/bench_qwen_tier46.json 2> /dev/null; echo "bench tier rc=$?"
      for lay in flashinfer_nhd flashinfer_hnd; do
        timeout 900 python bench.py --layout $lay --no-cpu-baseline --no-alt-modes > gpurun_out/bench_qwen_$lay.json 2> /dev/null; echo "bench $lay rc=$?"
      done
      for tp in 2 4 8; do
        timeout 900 python bench.py --workload llama70b32k --emulate-tp $tp --no-cpu-baseline > gpurun_out/bench_70b_tp$tp.json 2> /dev/null; echo "bench 70b tp$tp rc=$?"
        timeout 900 python bench.py --workload llama70b32k --emulate-tp $tp --mode zerocopy --no-cpu-baseline --no-hbm-arm --no-alt-modes > gpurun_out/bench_70b_tp${tp}_k1.json 2> /dev/null; echo "bench 70b tp$tp k1 rc=$?"
      done ;;
    tools)
      timeout 600 python tools/bench_queue.py > gpurun_out/bench_queue.json 2> /dev/null; echo "queue rc=$?"
      timeout 600 python tools/bench_peer.py > gpurun_out/peer_tier.jsonl 2> /dev/null; echo "peer rc=$?"
      timeout 900 python tools/bench_mixed.py > gpurun_out/bench_mixed_ref.json 2> /dev/null; echo "mixed rc=$?"
      timeout 900 python tools/bench_mixed.py --compute-per-token 4e-6 > gpurun_out/bench_mixed_b200.json 2> /dev/null; echo "mixed b200 rc=$?" ;;
    ncu)
      timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_bench_launches.csv \
        python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches rc=$?"
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ingest_ldg -s 40 -c 1 -o gpurun_out/prof_k2 \
        python bench.py --steps 1 --warmup 1 --no-cpu-baseline --workload llama8b32k > /dev/null 2>&1; echo "ncu k2 rc=$?"
      timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_chunk_digest|k_chain" -c 2 -o gpurun_out/prof_hash \
        python tools/prof_targets.py hash > /dev/null 2>&1; echo "ncu hash rc=$?"
      timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_score|k_tile_sort|k_merge_pass" -c 3 -o gpurun_out/prof_score \
        python tools/prof_targets.py scorer > /dev/null 2>&1; echo "ncu score rc=$?"
      timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ingest -c 1 -o gpurun_out/prof_k1 \
        python tools/prof_targets.py ingest-tp8 > /dev/null 2>&1; echo "ncu k1 rc=$?" ;;
  esac
done
