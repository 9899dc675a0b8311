import sys, json
sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import numpy as np, torch
from microbench import timed
from paper_2603_21257_b200 import hasher
for align in (1, 2, 4):
    rng = np.random.default_rng(0); n_req = 100_000
    lens = np.maximum(1, np.round(np.exp(np.log(28100) - 0.5 * np.log1p(0.25) + np.sqrt(np.log1p(0.25)) * rng.standard_normal(n_req)))).astype(np.int64)
    lens = (lens // align) * align + align
    offs = np.zeros(n_req + 1, np.int64); np.cumsum(lens, out=offs[1:])
    dev = torch.device("cuda")
    d_offs = torch.from_numpy(offs).to(dev)
    doc = torch.from_numpy(rng.integers(0, 1000, n_req)).to(dev); sh = torch.from_numpy(lens // 2).to(dev)
    tok = torch.empty(int(offs[-1]), dtype=torch.int32, device=dev)
    hasher.gen_tokens_device(0, d_offs, doc, sh, tok)
    coff = torch.from_numpy(hasher.chunk_offsets(offs)).to(dev)
    out = torch.empty(int(coff[-1]), dtype=torch.int64, device=dev)
    best, med = timed(lambda: hasher.hash_prefix_chunks_device(d_offs, tok, coff, out), reps=10)
    print(json.dumps(dict(align=align, ms=best * 1e3, GBps=(tok.numel() * 4 + out.numel() * 8) / best / 1e9)), flush=True)
    del tok, out
