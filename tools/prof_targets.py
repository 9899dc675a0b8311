"""Small, single-purpose workloads for ncu (one GPU, short):  python tools/prof_targets.py <what>

what: scorer | hash | index | ingest-ce | ingest-bulk | ingest-zerocopy | ingest-tp8 | ingest-hbm | ingest-hbm-tp8 |
      bulk-hbm | bulk-hbm-tp8 | bulk-hbm-tp8-hnd | ingest-ce-direct | ingest-hbm-tp4-hnd
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
from microbench import bench_hash, bench_scorer  # noqa: E402
from paper_2603_21257_b200 import ingest  # noqa: E402


def ingest_once(shape, n_chunks, mode, reps=2):
    pool = ingest.ChunkPool(shape, n_chunks)
    pool.fill_synthetic(3)
    l1 = ingest.PagedKVCache(shape, n_chunks * shape.pages_per_chunk, 1, n_chunks)
    cb = shape.page_bytes * shape.pages_per_chunk
    for c in range(n_chunks):
        g, row = l1.request(1, c, cb)
    l1.sync_block_table()
    items = ingest.items_numpy(np.arange(n_chunks), [row] * n_chunks, np.arange(n_chunks))
    evs = [torch.cuda.Event() for _ in range(shape.layers)]
    for _ in range(reps):
        ingest.ingest(l1, pool, items, mode=mode, layer_events=evs)
    torch.cuda.synchronize()
    assert ingest.verify_synthetic(l1, pool, items, 3) == 0


def ingest_hbm_bulk(shape, n_chunks, layout=0, reps=2):
    """K1b (tensor-map TMA) over an HBM-resident pool, whole layer range in one launch."""
    pool = ingest.ChunkPool.create_device(shape, n_chunks)
    pool.fill_synthetic(3)
    l1 = ingest.PagedKVCache(shape, n_chunks * shape.pages_per_chunk, 1, n_chunks, layout=layout)
    cb = shape.page_bytes * shape.pages_per_chunk
    for c in range(n_chunks):
        g, row = l1.request(1, c, cb)
    l1.sync_block_table()
    items = ingest.items_numpy(np.random.default_rng(0).permutation(n_chunks), [row] * n_chunks, np.arange(n_chunks))
    for _ in range(reps):
        ingest.ingest(l1, pool, items, mode=ingest.BULK)
    torch.cuda.synchronize()
    assert ingest.verify_synthetic(l1, pool, items, 3) == 0


def ingest_hbm(shape, n_chunks, reps=2, layout=0):
    """K1 over an HBM-resident pool as the stage issues it: layer 0 alone, then layers [1, L)."""
    pool = ingest.ChunkPool.create_device(shape, n_chunks)
    pool.fill_synthetic(3)
    l1 = ingest.PagedKVCache(shape, n_chunks * shape.pages_per_chunk, 1, n_chunks, layout=layout)
    cb = shape.page_bytes * shape.pages_per_chunk
    for c in range(n_chunks):
        g, row = l1.request(1, c, cb)
    l1.sync_block_table()
    items = ingest.items_numpy(np.random.default_rng(0).permutation(n_chunks), [row] * n_chunks, np.arange(n_chunks))
    evs = [torch.cuda.Event() if k in (0, shape.layers - 1) else None for k in range(shape.layers)]
    for _ in range(reps):
        ingest.ingest(l1, pool, items, layer_events=evs)
    torch.cuda.synchronize()
    assert ingest.verify_synthetic(l1, pool, items, 3) == 0


def index_once(n=4_000_000, n_req=100_000):
    """K7: insert n chunk hashes, then look up n_req requests' chunk lists (half of them hits)."""
    from paper_2603_21257_b200 import hasher

    rng = np.random.default_rng(0)
    keys = rng.integers(1, 2**63, n, dtype=np.int64).astype(np.uint64)
    idx = hasher.PrefixIndex(capacity=1 << 23)
    idx.insert(keys, np.arange(n, dtype=np.int64))
    per = n // n_req
    coffs = np.arange(n_req + 1, dtype=np.int64) * per
    probe = keys[: n_req * per].copy()
    probe[1::2] ^= np.uint64(1)  # misses from the second chunk of every other position
    idx.lookup(coffs, probe)
    torch.cuda.synchronize()


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "scorer":
        bench_scorer()
    elif what == "hash":
        bench_hash()
    elif what == "index":
        index_once()
    elif what == "ingest-ce":
        ingest_once(ingest.LLAMA31_8B, 128, ingest.CE)
    elif what == "ingest-bulk":
        ingest_once(ingest.LLAMA31_8B, 128, ingest.BULK)
    elif what == "ingest-zerocopy":
        ingest_once(ingest.LLAMA31_8B, 128, ingest.ZEROCOPY)
    elif what == "ingest-tp8":
        ingest_once(ingest.LLAMA3_70B.with_rank(8, 7), 128, ingest.ZEROCOPY)
    elif what == "ingest-hbm":
        ingest_hbm(ingest.LLAMA31_8B, 128)
    elif what == "bulk-hbm-tp8":
        ingest_hbm_bulk(ingest.LLAMA3_70B.with_rank(8, 7), 128)
    elif what == "bulk-hbm-tp8-hnd":
        ingest_hbm_bulk(ingest.LLAMA3_70B.with_rank(8, 7), 128, layout=ingest.LAYOUT_FLASHINFER_HND)
    elif what == "bulk-hbm":
        ingest_hbm_bulk(ingest.LLAMA31_8B, 128)
    elif what == "ingest-ce-direct":
        ingest_once(ingest.LLAMA31_8B, 128, ingest.CE_DIRECT)
    elif what == "ingest-hbm-tp8":
        ingest_hbm(ingest.LLAMA3_70B.with_rank(8, 7), 128)
    elif what == "ingest-hbm-tp4-hnd":
        ingest_hbm(ingest.LLAMA3_70B.with_rank(4, 1), 128, layout=ingest.LAYOUT_FLASHINFER_HND)
    else:
        raise SystemExit(__doc__)
