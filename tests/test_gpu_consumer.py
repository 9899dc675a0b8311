"""End-to-end layout proof: a real paged-attention consumer reads the pages the
ingest wrote.  FlashInfer's paged decode runs over l1.layer(l) through our block_table and must
match attention computed directly on the contiguous source chunks in the L2 pool."""
import numpy as np
import pytest
import torch

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

from paper_2603_21257_b200 import ingest  # noqa: E402
from paper_2603_21257_b200 import tiersim as t  # noqa: E402


def _reference_attention(q, k, v):
    """q [Hq, D], k/v [T, Hkv, D] (GQA): fp32 softmax attention."""
    hq, d = q.shape
    g = hq // k.shape[1]
    k = k.float().repeat_interleave(g, dim=1)  # [T, Hq, D]
    v = v.float().repeat_interleave(g, dim=1)
    s = torch.einsum("hd,thd->ht", q.float(), k) / d**0.5
    return torch.einsum("ht,thd->hd", torch.softmax(s, dim=-1), v)


@pytest.mark.parametrize("mode,layout", [("ce", "flash_attn"), ("bulk", "flash_attn"), ("ce", "flashinfer_nhd"),
                                         ("zerocopy", "flashinfer_nhd"), ("ce", "flashinfer_hnd"),
                                         ("zerocopy", "flashinfer_hnd")])
def test_flashinfer_paged_decode_reads_ingested_pages(mode, layout):
    """flash_attn: K and V planes passed as a (k, v) tuple; FlashInfer NHD / HND: the layer tensor
    [pages, 2, P, H, D] / [pages, 2, H, P, D] passed as is with kv_layout NHD / HND."""
    flashinfer = pytest.importorskip("flashinfer")
    shape = ingest.KVShape(layers=2, kv_heads=8, head_dim=128)
    pool = ingest.ChunkPool(shape, 12)
    pool.fill_synthetic(31)
    l1 = ingest.PagedKVCache(shape, num_pages=400, max_rows=4, max_chunks=8, layout=ingest.LAYOUTS[layout])
    cb = shape.page_bytes * shape.pages_per_chunk
    rng = np.random.default_rng(0)
    plans = {1: [5, 2, 9], 2: [0, 1], 3: [7, 8, 3, 11]}  # request -> pool slots of its chunks
    items, rows = [], {}
    for rid, slots in plans.items():
        for c, slot in enumerate(slots):
            granted, rows[rid] = l1.request(rid, c, cb)
            assert granted
            items.append((slot, rows[rid], c))
    l1.sync_block_table()
    ingest.ingest(l1, pool, ingest.items_numpy(*zip(*items)), mode=ingest.MODES[mode])
    torch.cuda.synchronize()

    bt = l1.block_table()
    indptr, indices, last = [0], [], []
    for rid, slots in plans.items():
        pages = bt[rows[rid], : len(slots) * 16]
        indices.extend(pages.tolist())
        indptr.append(len(indices))
        last.append(16)
    dev = torch.device("cuda")
    indptr_t = torch.tensor(indptr, dtype=torch.int32, device=dev)
    indices_t = torch.tensor(indices, dtype=torch.int32, device=dev)
    last_t = torch.tensor(last, dtype=torch.int32, device=dev)
    hq = 32
    chunks = torch.from_numpy(pool.slot_view(0, pool.n_slots).view(np.int16).copy()).view(torch.bfloat16)
    chunks = chunks.view(pool.n_slots, shape.layers, 2, 256, 8, 128)
    workspace = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
    for layer in range(shape.layers):
        kv = l1.layer(layer)
        kv_layout = "HND" if layout == "flashinfer_hnd" else "NHD"
        wrapper = flashinfer.BatchDecodeWithPagedKVCacheWrapper(workspace, kv_layout)
        wrapper.plan(indptr_t, indices_t, last_t, hq, 8, 128, 16, pos_encoding_mode="NONE",
                     q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
        q = (torch.randn(len(plans), hq, 128, generator=torch.Generator().manual_seed(layer)) * 0.05).to(dev, torch.bfloat16)
        out = wrapper.run(q, (kv[0], kv[1]) if layout == "flash_attn" else kv)
        for b, (rid, slots) in enumerate(plans.items()):
            src = chunks[slots, layer]  # [n_chunks, 2, 256, 8, 128]
            k = src[:, 0].reshape(-1, 8, 128).to(dev)
            v = src[:, 1].reshape(-1, 8, 128).to(dev)
            want = _reference_attention(q[b], k, v)
            torch.testing.assert_close(out[b].float(), want, atol=2e-2, rtol=2e-2)


@pytest.mark.parametrize("preplan", [True, False])
@pytest.mark.parametrize("layout", ["flash_attn", "flashinfer_nhd"])
def test_real_prefill_consumer_as_stage_hook(layout, preplan):
    """PagedPrefill (FlashInfer paged prefill + bf16 GEMMs per layer) runs as the stage's prefill
    hook, gated on per-layer fences: every page is verified, the consumer's last-layer attention
    equals attention over the source chunks, and ComputeDone follows residency.  preplan: attention
    planned before the run with the page list filled on device from the device block table (the
    default when every request has a wrapper), or planned at layer 0 from the host mirror."""
    pytest.importorskip("flashinfer")
    from paper_2603_21257_b200.consumer import PagedPrefill
    from paper_2603_21257_b200.stage import LoadStage

    shape = ingest.KVShape(layers=4, kv_heads=8, head_dim=128)
    pool = ingest.ChunkPool(shape, 16)
    pool.fill_synthetic(11)
    l1 = ingest.PagedKVCache(shape, 16 * 16, max_rows=4, max_chunks=16, layout=ingest.LAYOUTS[layout])
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(4, 8, 128, 2))
    q = t.QueueArrays(1, id=[5], arrival=[0.0], context_tokens=[256 * 6 + 100], query_tokens=[60],
                      cache_hit_ratio=[1.0], flags=np.zeros(1, np.uint8))
    slots = [[3, 9, 4, 0, 12, 7]]
    stage = LoadStage(l1, pool)
    cons = PagedPrefill(l1, q, cfg, hidden=1024, intermediate=2048, wrappers=2, preplan=preplan)
    assert cons.preplanned == preplan
    stage.set_prefill_hook(cons)
    res = stage.run(q, slots, cfg, prefill=True, layer_events=True, verify_seed=11)
    assert res.stats["verify_mismatches"] == 0 and cons.calls == shape.layers
    l1.sync_block_table()  # rows released at ComputeDone reach the device copy
    torch.cuda.synchronize()
    assert torch.equal(l1.block_table_device().cpu(), torch.from_numpy(l1.block_table().copy()))
    r = res.requests
    assert r["done_ms"][0] >= r["resident_ms"][0] >= r["first_layer_ms"][0]
    # the consumer's last layer: o = attention(q, cached K/V of layer L-1) -- against the source chunks
    ct = cons.ct[0]
    assert ct == 100 + 60
    chunks = torch.from_numpy(pool.slot_view(0, pool.n_slots).view(np.int16).copy()).view(torch.bfloat16)
    chunks = chunks.view(pool.n_slots, shape.layers, 2, 256, 8, 128)
    src = chunks[slots[0], shape.layers - 1]
    k = src[:, 0].reshape(-1, 8, 128).cuda()
    v = src[:, 1].reshape(-1, 8, 128).cuda()
    qs = cons.q_buf[:ct]
    for i in (0, 77, ct - 1):
        want = _reference_attention(qs[i], k, v)
        torch.testing.assert_close(cons.o_buf[i].float(), want, atol=2e-2, rtol=2e-2)
    # an exception in the hook fails the stage call with that exception
    def bad(*a):
        raise RuntimeError("consumer exploded")
    stage.set_prefill_hook(bad)
    with pytest.raises(RuntimeError, match="consumer exploded"):
        stage.run(q, slots, cfg, prefill=True)
    assert l1.reserved() == 0
