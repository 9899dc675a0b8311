#!/bin/bash
# Round-2 final evidence pass on one B200: the GPU suite, smoke, the contract bench line and the
# reference arm, the ncu launch list + --set full captures, compute-sanitizer.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_pytest_gpu.log 2>&1
echo "pytest -m gpu rc=$?"; tail -2 gpurun_out/final_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "bench ref rc=$?"
nproc > gpurun_out/final_platform.txt; lscpu | grep -E "Model name|NUMA|Socket|Thread|Core" >> gpurun_out/final_platform.txt
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit,pcie.link.gen.current,pcie.link.width.current --format=csv >> gpurun_out/final_platform.txt
bash tools/ncu_r02.sh
bash tools/sanitize_r02.sh
timeout 900 python bench.py --gpus 2 --one-device --workload llama70b32k --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final_bench_2rank_onedevice.json 2> gpurun_out/final_bench_2rank_onedevice.err; echo "2-rank one-device rc=$?"
