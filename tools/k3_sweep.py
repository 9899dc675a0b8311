"""K3 on the configs[4] queue (product generate_workload, loogle, 100K, seed 0): phase 1 alone and
phase 1 + chain, packed vs 16-byte-aligned request starts, 2-4 CTAs per SM, L2 prefetch distance.  CUDA events, mean of
10 after 3 warm-ups; against the 7.41 TB/s read-only ceiling.  One JSON line per case."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_21257_b200 import _capi, hasher  # noqa: E402
from paper_2603_21257_b200 import tiersim as t  # noqa: E402

CEIL = 7410.0
# (CTAs per SM, L2 prefetch distance in warp groups, chain fused into phase 1)
CASES = [(3, 1, 0), (3, 1, 1), (3, 0, 0), (3, 0, 1)]


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e-3 / reps


def main():
    q = t.generate_queue(t.WorkloadSpec(t.builtin_profile("loogle"), count=100_000, seed=0))
    lens = q.context_tokens
    n = len(lens)
    dev = torch.device("cuda")
    doc = torch.from_numpy(np.random.default_rng(1).integers(0, 1000, n)).to(dev)
    sh = torch.from_numpy(lens // 2).to(dev)
    coff = torch.from_numpy(hasher.chunk_offsets_of_lengths(lens)).to(dev)
    ref = None
    for layout in ("packed", "aligned"):
        if layout == "packed":
            offs = np.zeros(n + 1, np.int64)
            np.cumsum(lens, out=offs[1:])
        else:
            offs = hasher.aligned_offsets(lens)
        d_offs = torch.from_numpy(offs).to(dev)
        tok = torch.empty(int(offs[-1]), dtype=torch.int32, device=dev)
        hasher.gen_tokens_device(0, d_offs, doc, sh, tok)
        out = torch.empty(int(coff[-1]), dtype=torch.int64, device=dev)
        nbytes = int(lens.sum()) * 4 + out.numel() * 8
        for cps, pf, fused in CASES:
            t.check(_capi.lib.tsb_hash_set_grid(cps))
            t.check(_capi.lib.tsb_hash_set_tuning(pf, fused))
            p1 = timed(lambda: hasher.chunk_digests_device(d_offs, tok, coff, out))
            full = timed(lambda: hasher.hash_prefix_chunks_device(d_offs, tok, coff, out))
            h = out.cpu().numpy()
            ref = h if ref is None else ref
            print(json.dumps({"layout": layout, "ctas_per_sm": cps, "prefetch_groups": pf, "fused_chain": fused, "phase1_ms": p1 * 1e3, "total_ms": full * 1e3, "chain_ms": (full - p1) * 1e3,
                              "phase1_read_ceiling_frac": nbytes / p1 / 1e9 / CEIL,
                              "total_read_ceiling_frac": nbytes / full / 1e9 / CEIL,
                              "hashes_equal_first_case": bool(np.array_equal(h, ref))}), flush=True)
        del tok
    t.check(_capi.lib.tsb_hash_set_grid(0))
    t.check(_capi.lib.tsb_hash_set_tuning(1, 0))


if __name__ == "__main__":
    main()
