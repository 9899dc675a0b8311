"""K1 over an HBM-resident pool: sweep the grid for the stage's dominant launch shape (layers
[1, L) of one request); SHAPE=qwen|8b|70b|70b_tp2|70b_tp8.  One JSON line per grid."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_21257_b200 import ingest  # noqa: E402


def main():
    which = os.environ.get("SHAPE", "qwen")
    shape, n = {"qwen": (ingest.QWEN25_32B, 460), "8b": (ingest.LLAMA31_8B, 128),
                "70b": (ingest.LLAMA3_70B, 128), "70b_tp8": (ingest.LLAMA3_70B.with_rank(8, 3), 128),
                "70b_tp2": (ingest.LLAMA3_70B.with_rank(2, 1), 128)}[which]
    pool = ingest.ChunkPool.create_device(shape, n)
    pool.fill_synthetic(3)
    l1 = ingest.PagedKVCache(shape, n * shape.pages_per_chunk, 1, n)
    for c in range(n):
        g, row = l1.request(1, c, shape.page_bytes * shape.pages_per_chunk)
    l1.sync_block_table()
    items = ingest.items_numpy(np.random.default_rng(0).permutation(n), [row] * n, np.arange(n))
    dev_items = torch.from_numpy(items.view(np.uint8).copy()).cuda()
    s = torch.cuda.current_stream()
    alg = 2 * n * (shape.layers - 1) * 2 * 256 * shape.heads_local * 128 * 2
    for grid in [int(x) for x in sys.argv[1:]] or [296, 592, 888, 1184, 2368]:
        ingest.set_grid(0, 0, grid)
        f = lambda: ingest.ingest_device(l1, pool, dev_items, n, 1, shape.layers, mode=ingest.ZEROCOPY, stream=s)
        f()
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            f()
            b.record(s)
            b.synchronize()
            best = min(best, a.elapsed_time(b) * 1e-3)
        print(json.dumps(dict(shape=which, grid=grid, ms=best * 1e3,
                              TBps=alg / best / 1e12)), flush=True)
    ingest.set_grid()
    assert ingest.verify_synthetic(l1, pool, items, 3, 1, shape.layers) == 0


if __name__ == "__main__":
    main()
