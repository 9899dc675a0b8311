#!/bin/bash
# Round-2 first GPU pass: platform probes (topology, NUMA, host DRAM, TMA-tensor host reads), the GPU
# suite, the restructured bench (default + reference arm), and the multi-rank self-launch validation.
set -u
mkdir -p gpurun_out
{ nvidia-smi topo -m; nvidia-smi -q | grep -i -A3 "numa\|Bus Id" | head -30; lscpu | head -25;
  ls /sys/devices/system/node/; cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c; } > gpurun_out/platform.txt 2>&1
timeout 300 tools/probe/host_dram_probe 4096 > gpurun_out/host_dram_probe.jsonl 2>&1; echo "dram rc=$?"
timeout 600 tools/probe/tma_host_probe 4096 > gpurun_out/tma_host_probe.txt 2>&1; echo "tma rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest -m gpu rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
tail -c 600 gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench ref rc=$?"
timeout 900 python bench.py --gpus 2 --one-device --workload llama70b32k --steps 3 --warmup 3 --no-side --no-cpu-baseline \
  --no-hbm-tier > gpurun_out/bench_2rank_onedev.json 2> gpurun_out/bench_2rank_onedev.err; echo "bench 2rank rc=$?"
tail -c 600 gpurun_out/bench_2rank_onedev.err
timeout 900 python bench.py --pool hostalloc --steps 3 --warmup 2 --no-side --no-cpu-baseline --no-hbm-tier --no-alt-modes \
  > gpurun_out/bench_hostalloc.json 2> /dev/null; echo "bench hostalloc rc=$?"
