"""GPU: full-size parity at the BASELINE shapes, with checks that share no address math with the
ingest kernels.

  * a whole configs[1] request (Qwen2.5-32B KV, 128K @ 0.9 -> 460 chunks, 30.9 GB) and a configs[2]
    TP8 shard (Llama-3-70B KV, 32K, rank 3 of 8: 256-byte runs at a 2 KiB stride) are ingested
    through the public path (AUTO = copy engines + K2);
  * every word of every page is checked by k_verify_pages, which inverts the block table on the
    host and derives each word's source from the layout definition (verify.cu), not from
    seg_addr -- and is shown to be non-vacuous: one flipped word and one swapped block-table entry
    are caught with the exact expected counts;
  * sampled layers are compared byte for byte with the oracle's scatter_ref on the host.
"""
import numpy as np
import pytest
import torch

import pyoracle as po
from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

from paper_2603_21257_b200 import ingest  # noqa: E402

SEED = 90210


def ingest_request(shape, n_chunks, layout=ingest.LAYOUT_FLASH_ATTN, slot_order=None):
    pool = ingest.ChunkPool.create_numa(ingest.KVShape(shape.layers, shape.kv_heads, shape.head_dim), n_chunks,
                                        ingest.device_numa_node(0))
    pool.fill_synthetic(SEED)
    num_pages = n_chunks * shape.pages_per_chunk
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=2, max_chunks=n_chunks, layout=layout)
    cb = shape.page_bytes * shape.pages_per_chunk
    # a scrambled free list: pages of a chunk land far apart (exercise the block table)
    for c in range(n_chunks):
        g, row = l1.request(1, c, cb)
        assert g
    bt = l1.block_table()
    rng = np.random.default_rng(7)
    bt[row, :num_pages] = rng.permutation(num_pages).astype(np.int32)
    l1.sync_block_table()
    slots = np.arange(n_chunks) if slot_order is None else slot_order
    items = ingest.items_numpy(slots, [row] * n_chunks, np.arange(n_chunks))
    l1.arena.zero_()
    ingest.ingest(l1, pool, items)
    torch.cuda.synchronize()
    return pool, l1, items, row


def sampled_layers_equal(shape, pool, l1, items, layers, layout):
    view = pool.slot_view(0, pool.n_slots)
    bt = np.ascontiguousarray(l1.block_table())
    for lay in layers:
        want = po.scatter_ref_window(shape, view, items, bt, l1.num_pages, lay, lay + 1, threads=16, layout=layout)
        got = l1.arena[lay * l1.layer_bytes:(lay + 1) * l1.layer_bytes].cpu().numpy()
        assert np.array_equal(got, want), f"layer {lay} differs from scatter_ref"


def test_full_configs1_request_460_chunks():
    shape = ingest.QWEN25_32B
    pool, l1, items, row = ingest_request(shape, 460)
    assert ingest.verify_synthetic(l1, pool, items, SEED) == 0
    sampled_layers_equal(shape, pool, l1, items, (0, 31, 63), ingest.LAYOUT_FLASH_ATTN)
    # non-vacuous: one flipped word -> exactly one mismatch; two swapped pages -> both pages wrong
    l1.arena[l1.layer_bytes * 17 + 12345 * 8] ^= 0x5A
    assert ingest.verify_synthetic(l1, pool, items, SEED) == 1
    l1.arena[l1.layer_bytes * 17 + 12345 * 8] ^= 0x5A
    bt = l1.block_table()
    a, b = int(bt[row, 5]), int(bt[row, 900])
    bt[row, 5], bt[row, 900] = b, a
    words_per_page = shape.layers * 2 * 16 * 8 * 128 * 2 // 8
    assert ingest.verify_synthetic(l1, pool, items, SEED) == 2 * words_per_page
    bt[row, 5], bt[row, 900] = a, b
    assert ingest.verify_synthetic(l1, pool, items, SEED) == 0


@pytest.mark.parametrize("layout", [ingest.LAYOUT_FLASH_ATTN, ingest.LAYOUT_FLASHINFER_HND])
def test_full_configs2_tp8_shard(layout):
    shape = ingest.LLAMA3_70B.with_rank(8, 3)
    order = np.random.default_rng(3).permutation(128)  # scattered slots
    pool, l1, items, row = ingest_request(shape, 128, layout=layout, slot_order=order)
    assert ingest.verify_synthetic(l1, pool, items, SEED) == 0
    sampled_layers_equal(shape, pool, l1, items, (0, 40, 79), layout)
    # the same pages read as rank 2's heads must fail everywhere (the head offset is checked)
    other = ingest.PagedKVCache(ingest.LLAMA3_70B.with_rank(8, 2), l1.num_pages, max_rows=2, max_chunks=128,
                                arena=l1.arena, layout=layout)
    cb = other.shape.page_bytes * other.shape.pages_per_chunk
    for c in range(128):
        other.request(1, c, cb)
    other.block_table()[:] = l1.block_table()
    assert ingest.verify_synthetic(other, pool, items, SEED) == 128 * 16 * 80 * 2 * 16 * 128 * 2 // 8
