#!/bin/bash
# Round 2: CE-direct with strip-merged 2D copies -- parity, per-fence rates, the stage A/B again.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stage_random.py tests/test_gpu_stage.py -q -p no:cacheprovider -x > gpurun_out/cd_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/cd_pytest.log
timeout 300 python tools/probe/overlap_probe.py > gpurun_out/cd_overlap_probe.jsonl 2>&1; echo "overlap rc=$?"; cat gpurun_out/cd_overlap_probe.jsonl
for m in auto ce_direct; do
  timeout 900 python tools/bench_mixed.py --compute-per-token 4e-6 --mode $m > gpurun_out/cd_mixed_k6_${m}.json 2> /dev/null; echo "k6 $m rc=$?"
  timeout 900 python tools/bench_mixed.py --consumer real --n 24 --mode $m > gpurun_out/cd_mixed_real_${m}.json 2> /dev/null; echo "real $m rc=$?"
done
