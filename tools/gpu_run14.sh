mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/bench_queue.py > gpurun_out/bench_queue.json 2>/dev/null; echo "q rc=$?"
timeout 900 python tools/bench_mixed.py > gpurun_out/bench_mixed_ref.json 2>/dev/null; echo "m1 rc=$?"
timeout 900 python tools/bench_mixed.py --compute-per-token 4e-6 > gpurun_out/bench_mixed_b200.json 2>/dev/null; echo "m2 rc=$?"
timeout 900 python bench.py > gpurun_out/bench_default.json 2>/dev/null; echo "b rc=$?"
timeout 900 python bench.py --workload llama70b32k --mode zerocopy > gpurun_out/bench_70b.json 2>/dev/null; echo "b70 rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2>/dev/null; echo "ref rc=$?"
