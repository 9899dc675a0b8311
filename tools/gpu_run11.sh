mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "order or scores or scheduler or deadline or signed" 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_scorer_launches.csv python tools/prof_targets.py scorer 2>&1 | grep "^{"
