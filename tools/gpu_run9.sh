set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python tools/bench_queue.py > gpurun_out/bench_queue.json 2> gpurun_out/bench_queue.err; echo "q rc=$?"; cat gpurun_out/bench_queue.json; tail -3 gpurun_out/bench_queue.err
timeout 900 python tools/bench_mixed.py > gpurun_out/bench_mixed.json 2> gpurun_out/bench_mixed.err; echo "m rc=$?"; cat gpurun_out/bench_mixed.json; tail -3 gpurun_out/bench_mixed.err
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "b rc=$?"; cat gpurun_out/bench_default.json; grep -v CUDAEvent gpurun_out/bench_default.err | tail -3
