"""One K3 pass on the configs[4] queue (aligned layout) for ncu: `python tools/prof_k3.py PF FUSED`."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_21257_b200 import _capi, hasher  # noqa: E402
from paper_2603_21257_b200 import tiersim as t  # noqa: E402

pf, fused = int(sys.argv[1]), int(sys.argv[2])
q = t.generate_queue(t.WorkloadSpec(t.builtin_profile("loogle"), count=100_000, seed=0))
lens = q.context_tokens
n = len(lens)
dev = torch.device("cuda")
offs = hasher.aligned_offsets(lens)
d_offs = torch.from_numpy(offs).to(dev)
tok = torch.empty(int(offs[-1]), dtype=torch.int32, device=dev)
hasher.gen_tokens_device(0, d_offs, torch.from_numpy(np.random.default_rng(1).integers(0, 1000, n)).to(dev),
                         torch.from_numpy(lens // 2).to(dev), tok)
coff = torch.from_numpy(hasher.chunk_offsets_of_lengths(lens)).to(dev)
out = torch.empty(int(coff[-1]), dtype=torch.int64, device=dev)
t.check(_capi.lib.tsb_hash_set_tuning(pf, fused))
for _ in range(2):
    hasher.hash_prefix_chunks_device(d_offs, tok, coff, out)
torch.cuda.synchronize()
