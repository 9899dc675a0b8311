set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "k2_scatter or ce_copy" 2>&1 | tail -3
timeout 600 python bench.py --workload llama8b32k --steps 3 --warmup 3 > gpurun_out/bench_llama8b.json 2> gpurun_out/bench_llama8b.err; echo "b1 rc=$?"; cat gpurun_out/bench_llama8b.json; grep -v CUDAEvent gpurun_out/bench_llama8b.err | tail -5
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "b2 rc=$?"; cat gpurun_out/bench_default.json; grep -v CUDAEvent gpurun_out/bench_default.err | tail -5
