mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_consumer.py -q -p no:cacheprovider -x 2>&1 | tail -30
