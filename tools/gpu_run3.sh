set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "
import sys; sys.argv=['x']; sys.path.insert(0,'tools')
from microbench import bench_hash, bench_ingest
from paper_2603_21257_b200 import ingest
import numpy as np
bench_hash()
bench_ingest(ingest.LLAMA31_8B, 128, ['ce'], per_layer=True, ce_variants=(1,2), slots=np.random.default_rng(0).permutation(128))
" 2>&1 | grep "^{"
