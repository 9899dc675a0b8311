mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "hash" 2>&1 | tail -2
timeout 300 python -c "
import sys; sys.argv=['x']; sys.path.insert(0,'tools')
from microbench import bench_hash
bench_hash(); bench_hash()
" 2>&1 | grep "^{"
timeout 600 ncu --set full --clock-control none -k regex:"k_chunk_digest|k_chain" -c 2 -o gpurun_out/prof_hash3 python tools/prof_targets.py hash > /dev/null 2>&1; echo "ncu rc=$?"
