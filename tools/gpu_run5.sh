set -x
mkdir -p gpurun_out
df -h /dev/shm; free -g
timeout 600 python bench.py --workload llama8b32k --steps 3 --warmup 3 > gpurun_out/bench_llama8b.json 2> gpurun_out/bench_llama8b.err; echo "b1 rc=$?"; cat gpurun_out/bench_llama8b.json; tail -5 gpurun_out/bench_llama8b.err
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "b2 rc=$?"; cat gpurun_out/bench_default.json; tail -5 gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "b3 rc=$?"; cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
