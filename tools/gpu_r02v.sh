#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_stage_modes.py tests/test_gpu_stage_random.py -q -p no:cacheprovider -x 2>&1 | tail -15
