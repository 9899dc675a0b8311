"""Randomised end-to-end stage runs (GPU): random KV geometry (layers, heads, head_dim, fp8/bf16,
chunk and page sizes), TP shard, page layout, ingest mode, policy, L1 pressure and HBM-tier
chunks.  Every run must verify every page against the synthetic source, move exactly the planned
bytes, release every page, and admit requests in the oracle's pick order."""
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
import pyoracle as po  # noqa: E402

from paper_2603_21257_b200 import ingest  # noqa: E402
from paper_2603_21257_b200 import tiersim as t  # noqa: E402
from paper_2603_21257_b200.stage import LoadStage  # noqa: E402

# TSB_SOAK=N widens both sweeps N-fold (a soak run; the default keeps the suite at ~1 minute)
SOAK = max(1, int(__import__("os").environ.get("TSB_SOAK", "1")))


def _case(seed):
    rng = np.random.default_rng(seed)
    heads = int(rng.choice([1, 2, 4, 8]))
    tp = int(rng.choice([d for d in (1, 2, 4, 8) if heads % d == 0]))
    chunk = int(rng.choice([64, 128, 256]))
    page = int(rng.choice([p for p in (8, 16, 32) if chunk % p == 0]))
    full = ingest.KVShape(layers=int(rng.integers(1, 5)), kv_heads=heads, head_dim=int(rng.choice([64, 128])),
                          dtype_bytes=int(rng.choice([1, 2])), chunk_tokens=chunk, page_tokens=page)
    shape = full.with_rank(tp, int(rng.integers(tp)))
    layout = int(rng.integers(3))
    modes = ["auto", "ce", "zerocopy", "bulk"] + (["ce_direct"] if tp == 1 and layout != 2 else [])
    return rng, full, shape, layout, str(rng.choice(modes)), int(rng.integers(5))


@pytest.mark.parametrize("seed", range(64 * SOAK))
def test_random_stage_runs_verify(seed):
    rng, full, shape, layout, mode, policy = _case(seed)
    n_slots = int(rng.integers(4, 12))
    pool = ingest.ChunkPool(full, n_slots)
    pool.fill_synthetic(1000 + seed)
    tier = None
    if rng.random() < 0.5:
        tier = ingest.ChunkPool.create_device(full, n_slots)
        tier.fill_synthetic(1000 + seed)  # same content per slot index as the host pool
    n = int(rng.integers(1, 7))
    chunks = rng.integers(0, 6, n)
    query = rng.integers(1, 50, n)
    ctx = chunks * full.chunk_tokens + rng.integers(0, full.chunk_tokens, n)
    q = t.QueueArrays(n, id=rng.permutation(n) + 10, arrival=np.round(rng.random(n), 2), context_tokens=ctx,
                      query_tokens=query, cache_hit_ratio=np.ones(n), flags=np.full(n, 1, np.uint8),
                      deadline=1.0 + rng.random(n))
    slot_lists = []
    for i in range(n):
        nb = int(np.floor(ctx[i] * 1.0 / full.chunk_tokens))
        sl = [int(rng.integers(n_slots)) for _ in range(nb)]
        if tier is not None:
            sl = [~s if rng.random() < 0.4 else s for s in sl]
        slot_lists.append(sl)
    max_nb = max([len(s) for s in slot_lists] + [1])
    ppc = shape.pages_per_chunk
    num_pages = int(ppc * (max_nb + rng.integers(0, 8)))  # at least the largest request: deferral, never deadlock
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=n + 1, max_chunks=max_nb, layout=layout)
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(full.layers, full.kv_heads, full.head_dim,
                                                               full.dtype_bytes),
                          block_size_tokens=full.chunk_tokens)
    stage = LoadStage(l1, pool)
    if tier is not None:
        stage.set_hbm_tier(tier)
    res = stage.run(q, slot_lists, cfg, policy=policy, mode=ingest.MODES[mode], verify_seed=1000 + seed,
                    layer_events=bool(rng.integers(2)))
    torch.cuda.synchronize()
    assert res.stats["verify_mismatches"] == 0, (seed, mode, layout)
    assert res.stats["bytes"] == sum(len(s) for s in slot_lists) * shape.local_chunk_bytes
    assert l1.reserved() == 0 and l1.free_pages() == num_pages
    m = t.cost_models_from_config(cfg)
    st, _, _, _, pr = po.score_queue(q, policy, [m.load.slope, m.load.intercept, m.comp.slope, m.comp.intercept], cfg)
    assert st == 0
    want = po.sort_order(pr, q.arrival, q.id)
    assert list(np.argsort(res.requests["pick_position"])) == list(want)
    # the same batch with reuse_l1 (K8 replication from live holders) and a K6 prefill sharing the GPU
    # (AUTO resolves per call as without the prefill: CE + K2 for host pools)
    res2 = stage.run(q, slot_lists, cfg, policy=policy, verify_seed=1000 + seed, reuse_l1=True, prefill=True,
                     layer_events=bool(seed % 2))
    assert res2.stats["verify_mismatches"] == 0, (seed, "reuse", layout)
    assert res2.stats["bytes"] == res.stats["bytes"]
    assert l1.reserved() == 0 and l1.free_pages() == num_pages


@pytest.mark.parametrize("seed", range(12 * SOAK))
def test_random_online_runs_verify(seed):
    """The real-time loop (tsb_stage_run_online) over random geometries, layouts and HBM-tier
    chunks: arrivals within ~20 ms, prefill burner on; every page verified before release."""
    rng, full, shape, layout, mode, policy = _case(100 + seed)
    n_slots = int(rng.integers(4, 10))
    pool = ingest.ChunkPool(full, n_slots)
    pool.fill_synthetic(7 + seed)
    tier = ingest.ChunkPool.create_device(full, n_slots)
    tier.fill_synthetic(7 + seed)
    n = int(rng.integers(2, 7))
    ctx = rng.integers(1, 5, n) * full.chunk_tokens
    q = t.QueueArrays(n, id=np.arange(n) + 1, arrival=np.sort(np.round(rng.random(n) * 0.02, 4)),
                      context_tokens=ctx, query_tokens=np.full(n, 8), cache_hit_ratio=np.ones(n),
                      flags=np.full(n, 1, np.uint8), deadline=0.5 + rng.random(n))
    slot_lists = [[(~s if rng.random() < 0.3 else s) for s in rng.integers(0, n_slots, int(c // full.chunk_tokens))]
                  for c in ctx]
    ppc = shape.pages_per_chunk
    l1 = ingest.PagedKVCache(shape, int(ppc * (4 + rng.integers(0, 4))), max_rows=n + 1, max_chunks=4,
                             layout=layout)
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(full.layers, full.kv_heads, full.head_dim,
                                                               full.dtype_bytes),
                          block_size_tokens=full.chunk_tokens, compute_per_token=1e-7, compute_base=1e-4)
    stage = LoadStage(l1, pool)
    stage.set_hbm_tier(tier)
    res = stage.run_online(q, slot_lists, cfg, policy=policy, mode=ingest.MODES[mode], verify_seed=7 + seed)
    assert res.stats["verify_mismatches"] == 0, (seed, mode, layout)
    assert res.stats["bytes"] == sum(len(s) for s in slot_lists) * shape.local_chunk_bytes
    assert l1.reserved() == 0
    # the same replay with reuse_l1 (host-pool chunks replicated from live holders by K8)
    res2 = stage.run_online(q, slot_lists, cfg, policy=policy, mode=ingest.MODES[mode], verify_seed=7 + seed,
                            reuse_l1=True)
    assert res2.stats["verify_mismatches"] == 0, (seed, "reuse", mode, layout)
    assert res2.stats["bytes"] == res.stats["bytes"]
    assert l1.reserved() == 0 and l1.free_pages() == l1.num_pages
