mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stage.py tests/test_cpp_api.py -q -p no:cacheprovider -x 2>&1 | tail -5
timeout 900 python tools/bench_online.py > gpurun_out/bench_online.json 2> gpurun_out/bench_online.err; echo "online rc=$?"; tail -8 gpurun_out/bench_online.err
