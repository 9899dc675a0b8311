set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python tools/bench_queue.py > gpurun_out/bench_queue.json 2> gpurun_out/bench_queue.err; echo "q rc=$?"; cat gpurun_out/bench_queue.json; tail -3 gpurun_out/bench_queue.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_scorer_launches.csv python tools/prof_targets.py scorer > /dev/null 2>&1; echo "ncu rc=$?"
