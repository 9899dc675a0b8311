set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "
import sys; sys.argv=['x']; sys.path.insert(0,'tools')
from microbench import bench_hash
bench_hash()
" 2>&1 | grep "^{"
