"""Exploratory device-timed microbenchmarks (not the contract bench; see bench.py).

python tools/microbench.py [--quick]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_21257_b200 import hasher, ingest  # noqa: E402
from paper_2603_21257_b200 import tiersim as t  # noqa: E402
from paper_2603_21257_b200.scorer import BatchScorer, DeviceQueue  # noqa: E402


def timed(fn, reps=5, warm=2, stream=None):
    s = stream or torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return min(ts), float(np.median(ts))


def bench_ingest(shape, n_chunks, modes, per_layer, grids=None, ce_variants=(1,), slots=None):
    res = []
    pool = ingest.ChunkPool(shape, n_chunks)
    pool.fill_synthetic(3)
    l1 = ingest.PagedKVCache(shape, n_chunks * shape.pages_per_chunk, 1, n_chunks)
    cb = shape.page_bytes * shape.pages_per_chunk
    for c in range(n_chunks):
        g, row = l1.request(1, c, cb)
    l1.sync_block_table()
    src = np.arange(n_chunks) if slots is None else slots
    items = ingest.items_numpy(src, [row] * n_chunks, np.arange(n_chunks))
    payload = n_chunks * shape.local_chunk_bytes
    evs = [torch.cuda.Event() for _ in range(shape.layers)] if per_layer else None
    for mode in modes:
        for g in (grids or [0]):
            for v in (ce_variants if mode == "ce" else (1,)):
                ingest.set_grid(zerocopy_ctas=g if mode == "zerocopy" else 0, bulk_ctas=g if mode == "bulk" else 0)
                ingest.set_ce(v)
                m = ingest.MODES[mode]
                fn = lambda: ingest.ingest(l1, pool, items, mode=m, layer_events=evs)
                best, med = timed(fn, reps=3, warm=1)
                ok = ingest.verify_synthetic(l1, pool, items, 3)
                res.append(dict(shape=f"L{shape.layers}H{shape.kv_heads}tp{shape.tp_size}", chunks=n_chunks,
                                mode=mode, ce_variant=v, grid=g, per_layer=per_layer, GBps=payload / best / 1e9,
                                med_GBps=payload / med / 1e9, mismatches=ok))
                print(json.dumps(res[-1]), flush=True)
    ingest.set_grid()
    ingest.set_ce()
    pool.close()
    l1.close()
    return res


def bench_ce_peak():
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    best, _ = timed(lambda: d.copy_(h, non_blocking=True), reps=5)
    print(json.dumps(dict(ce_h2d_GBps=n / best / 1e9)), flush=True)


def bench_scorer(n=100_000):
    rng = np.random.default_rng(0)
    q = t.QueueArrays(n, id=np.arange(n), arrival=np.cumsum(rng.exponential(0.5, n)),
                      context_tokens=rng.integers(2000, 128000, n), query_tokens=rng.integers(1, 300, n),
                      cache_hit_ratio=rng.choice([0.25, 0.5, 0.75, 0.9, 1.0], n), flags=np.ones(n, np.uint8),
                      deadline=np.cumsum(rng.exponential(0.5, n)) + 10)
    dq = DeviceQueue(q)
    sc = BatchScorer(0)
    cfg = t.ClusterConfig()
    m = t.cost_models_from_config(cfg)
    out = sc.score_device(dq, 4, m, cfg)
    for pol in range(5):
        best, med = timed(lambda: sc.score_device(dq, pol, m, cfg, out=out, check_errors=False), reps=20, warm=3)
        print(json.dumps(dict(scorer_policy=pol, n=n, us=best * 1e6, med_us=med * 1e6)), flush=True)
    best, _ = timed(lambda: sc.score(q, 4, m, cfg), reps=5)
    print(json.dumps(dict(scorer_host_e2e_us=best * 1e6)), flush=True)


def bench_hash(n_req=100_000):
    rng = np.random.default_rng(0)
    lens = np.maximum(1, np.round(np.exp(np.log(28100) - 0.5 * np.log1p(0.25) +
                                         np.sqrt(np.log1p(0.25)) * rng.standard_normal(n_req)))).astype(np.int64)
    offs = np.zeros(n_req + 1, np.int64)
    np.cumsum(lens, out=offs[1:])
    dev = torch.device("cuda")
    d_offs = torch.from_numpy(offs).to(dev)
    doc = torch.from_numpy(rng.integers(0, 1000, n_req)).to(dev)
    sh = torch.from_numpy(lens // 2).to(dev)
    tok = torch.empty(int(offs[-1]), dtype=torch.int32, device=dev)
    hasher.gen_tokens_device(0, d_offs, doc, sh, tok)
    coff = torch.from_numpy(hasher.chunk_offsets(offs)).to(dev)
    out = torch.empty(int(coff[-1]), dtype=torch.int64, device=dev)
    best, med = timed(lambda: hasher.hash_prefix_chunks_device(d_offs, tok, coff, out), reps=10)
    nbytes = tok.numel() * 4 + out.numel() * 8
    print(json.dumps(dict(hash_tokens=int(offs[-1]), chunks=int(coff[-1]), ms=best * 1e3, GBps=nbytes / best / 1e9)),
          flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    bench_ce_peak()
    bench_ingest(ingest.LLAMA31_8B, 128, ["ce"], per_layer=True, ce_variants=(0, 1))
    bench_ingest(ingest.LLAMA31_8B, 128, ["ce"], per_layer=True, ce_variants=(0, 1),
                 slots=np.random.default_rng(0).permutation(128))
    bench_ingest(ingest.LLAMA31_8B, 128, ["bulk", "zerocopy", "ce"], per_layer=False)
    bench_ingest(ingest.QWEN25_32B, 460, ["ce", "bulk"], per_layer=True)
    for tp in (2, 4, 8):
        shp = ingest.LLAMA3_70B.with_rank(tp, tp - 1)
        bench_ingest(shp, 128, ["bulk", "zerocopy"], per_layer=True, grids=[32, 64, 128])
    if not a.quick:
        bench_scorer()
        bench_hash()
