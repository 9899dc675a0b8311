"""GPU: the L2 chunk index (K7) against a dict-based restatement, and the full
request path: tokens -> prefix hashes (K3) -> index lookup (K7) -> load stage over the matched
slots -> pages verified."""
import numpy as np
import pytest

import pyoracle as po
from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

from paper_2603_21257_b200 import hasher, ingest  # noqa: E402
from paper_2603_21257_b200 import tiersim as t  # noqa: E402
from paper_2603_21257_b200.stage import LoadStage  # noqa: E402


def lookup_ref(index: dict, coffs, hashes):
    """Restatement: matched = leading chunks whose hash is indexed; slots -1 from the first miss."""
    matched, slots = [], np.full(len(hashes), -1, np.int64)
    for r in range(len(coffs) - 1):
        m = 0
        for c in range(coffs[r], coffs[r + 1]):
            if hashes[c] not in index:
                break
            slots[c] = index[hashes[c]]
            m += 1
        matched.append(m)
    return np.array(matched, np.int64), slots


def test_index_lookup_matches_dict_restatement():
    rng = np.random.default_rng(0)
    # documents (stored in L2) and requests that share prefixes of them, then diverge
    docs = {d: int(rng.integers(4, 40)) * 256 for d in range(12)}
    doff = np.zeros(len(docs) + 1, np.int64)
    np.cumsum(list(docs.values()), out=doff[1:])
    dtok = po.gen_tokens(7, doff, np.arange(len(docs)), np.array(list(docs.values())))
    dh = po.hash_prefix_chunks(doff, dtok)
    dco = hasher.chunk_offsets(doff)
    index = {}
    slots_of_doc = np.arange(len(dh), dtype=np.int64) + 1000
    for d in range(len(docs)):
        if d % 4 == 3:
            continue  # documents never stored: requests over them miss from chunk 0
        for c in range(dco[d], dco[d + 1]):
            index[int(dh[c])] = int(slots_of_doc[c])
    idx = hasher.PrefixIndex(capacity=4 * len(dh))
    keep = np.array([(c >= dco[d] and c < dco[d + 1] and d % 4 != 3) for d in range(len(docs))
                     for c in range(dco[d], dco[d + 1])])
    idx.insert(dh[keep], slots_of_doc[keep])
    live, full = idx.stats()
    assert live == keep.sum() and full == 0
    # 200 requests: doc prefix of random length (possibly beyond the doc), then their own tokens
    n = 200
    doc = rng.integers(0, len(docs), n)
    shared = np.array([int(rng.integers(0, docs[d] + 600)) for d in doc])
    lens = shared + rng.integers(0, 3000, n)
    offs = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=offs[1:])
    # tokens past a document's end come from the request's own stream: emulate by capping shared
    shared = np.minimum(shared, [docs[d] for d in doc])
    toks = po.gen_tokens(7, offs, doc, shared)
    hashes = hasher.hash_prefix_chunks(offs, toks)
    coffs = hasher.chunk_offsets(offs)
    m, s = idx.lookup(coffs, hashes)
    want_m, want_s = lookup_ref(index, coffs, [int(h) for h in hashes])
    assert np.array_equal(m, want_m) and np.array_equal(s, want_s)
    assert 0 < m.sum() < len(hashes)  # both hits and misses exercised
    # erase a document's chunks: lookups now stop before them
    import torch

    gone = dh[dco[0]:dco[1]]
    idx.erase_device(torch.from_numpy(gone.view(np.int64)).cuda())
    for h in gone:
        index.pop(int(h), None)
    m2, s2 = idx.lookup(coffs, hashes)
    want_m2, want_s2 = lookup_ref(index, coffs, [int(h) for h in hashes])
    assert np.array_equal(m2, want_m2) and np.array_equal(s2, want_s2)


def test_request_path_tokens_to_pages():
    """tokens -> K3 hashes -> K7 matched prefix + slots -> stage ingest -> pages verified."""
    shape = ingest.KVShape(layers=2, kv_heads=8, head_dim=128)
    n_docs, doc_chunks = 3, 24
    pool = ingest.ChunkPool(shape, n_docs * doc_chunks)
    pool.fill_synthetic(13)
    doff = np.arange(n_docs + 1, dtype=np.int64) * doc_chunks * 256
    dtok = po.gen_tokens(3, doff, np.arange(n_docs), np.full(n_docs, doc_chunks * 256))
    dh = hasher.hash_prefix_chunks(doff, dtok)
    idx = hasher.PrefixIndex(capacity=1024)
    idx.insert(dh, np.arange(len(dh)))  # L2: doc d chunk c at slot d*24 + c
    # requests: question over doc d, sharing k*256 + partial tokens
    n = 6
    doc = np.array([0, 1, 2, 0, 1, 2])
    shared = np.array([24 * 256, 10 * 256 + 100, 5 * 256, 3 * 256 + 255, 0, 24 * 256])
    lens = shared + 500
    offs = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=offs[1:])
    toks = po.gen_tokens(3, offs, doc, shared)
    hashes = hasher.hash_prefix_chunks(offs, toks)
    coffs = hasher.chunk_offsets(offs)
    matched, slots = idx.lookup(coffs, hashes)
    assert list(matched) == [24, 10, 5, 3, 0, 24]
    q = t.QueueArrays(n, id=np.arange(1, n + 1), arrival=np.arange(n) * 0.1, context_tokens=lens,
                      query_tokens=np.full(n, 20),
                      cache_hit_ratio=[hasher.hit_ratio_for_match(int(lens[i]), int(matched[i])) for i in range(n)],
                      flags=np.zeros(n, np.uint8))
    slot_lists = [list(slots[coffs[i]:coffs[i] + matched[i]]) for i in range(n)]
    assert all(s == doc[i] * 24 + c for i in range(n) for c, s in enumerate(slot_lists[i]))
    l1 = ingest.PagedKVCache(shape, 40 * 16, max_rows=8, max_chunks=32)
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(2, 8, 128, 2))
    res = LoadStage(l1, pool).run(q, slot_lists, cfg, verify_seed=13)
    assert res.stats["verify_mismatches"] == 0
    assert list(res.requests["chunks"]) == list(matched)


def test_request_path_with_hbm_tier_hits():
    """The index stores ~slot for chunks resident in the HBM tier: lookups hand the stage negative
    slots, which tsb_stage_set_hbm_tier routes to the tier; every page still verifies."""
    shape = ingest.KVShape(layers=2, kv_heads=8, head_dim=128)
    n_docs, doc_chunks = 2, 16
    pool = ingest.ChunkPool(shape, n_docs * doc_chunks)
    pool.fill_synthetic(19)
    tier = ingest.ChunkPool.create_device(shape, n_docs * doc_chunks)
    tier.fill_synthetic(19)  # same content per slot index
    doff = np.arange(n_docs + 1, dtype=np.int64) * doc_chunks * 256
    dtok = po.gen_tokens(4, doff, np.arange(n_docs), np.full(n_docs, doc_chunks * 256))
    dh = hasher.hash_prefix_chunks(doff, dtok)
    vals = np.arange(len(dh), dtype=np.int64)
    hot = (vals % doc_chunks) < 6  # the first 6 chunks of every document are in the HBM tier
    vals[hot] = ~vals[hot]
    idx = hasher.PrefixIndex(capacity=256)
    idx.insert(dh, vals)
    n = 4
    doc = np.array([0, 1, 0, 1])
    shared = np.array([16 * 256, 9 * 256 + 7, 4 * 256, 0])
    lens = shared + 300
    offs = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=offs[1:])
    toks = po.gen_tokens(4, offs, doc, shared)
    coffs = hasher.chunk_offsets(offs)
    matched, slots = idx.lookup(coffs, hasher.hash_prefix_chunks(offs, toks))
    assert list(matched) == [16, 9, 4, 0]
    slot_lists = [list(slots[coffs[i]:coffs[i] + matched[i]]) for i in range(n)]
    assert slot_lists[0][:6] == [~c for c in range(6)] and slot_lists[0][6] == 6
    q = t.QueueArrays(n, id=np.arange(1, n + 1), arrival=np.arange(n) * 0.1, context_tokens=lens,
                      query_tokens=np.full(n, 20),
                      cache_hit_ratio=[hasher.hit_ratio_for_match(int(lens[i]), int(matched[i])) for i in range(n)],
                      flags=np.zeros(n, np.uint8))
    l1 = ingest.PagedKVCache(shape, 20 * 16, max_rows=8, max_chunks=32)
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(2, 8, 128, 2))
    stage = LoadStage(l1, pool)
    stage.set_hbm_tier(tier)
    res = stage.run(q, slot_lists, cfg, verify_seed=19)
    assert res.stats["verify_mismatches"] == 0
    assert list(res.requests["chunks"]) == list(matched)


def test_duplicate_keys_in_one_batch_resolve_to_the_lowest_index():
    """LooGLE-like batches index the same document chunk from several requests at once: the entry
    must hold the value of the FIRST occurrence in the batch, every time (no race)."""
    rng = np.random.default_rng(5)
    uniq = rng.integers(1, 2**62, 3000).astype(np.uint64)
    reps = rng.integers(0, len(uniq), 60000)
    keys = uniq[reps]
    vals = np.arange(len(keys), dtype=np.int64) + 7
    first = {}
    for i, k in enumerate(keys.tolist()):
        first.setdefault(k, int(vals[i]))
    for trial in range(5):
        idx = hasher.PrefixIndex(capacity=1 << 13)
        perm = rng.permutation(len(keys)) if trial else np.arange(len(keys))
        idx.insert(keys[perm], vals[perm])
        want = {}
        for i in perm.tolist():
            want.setdefault(int(keys[i]), int(vals[i]))
        co = np.arange(len(uniq) + 1, dtype=np.int64)
        m, got = idx.lookup(co, uniq)
        assert np.all(m == 1)
        assert [want[int(k)] for k in uniq.tolist()] == got.tolist()
        assert idx.stats() == (len(uniq), 0)
        # a later batch re-indexes: the newest call wins, again lowest index within it
        idx.insert(keys[:10], vals[:10] + 10**9)
        m, got2 = idx.lookup(np.arange(11, dtype=np.int64), keys[:10])
        firsts = {}
        for i in range(10):
            firsts.setdefault(int(keys[i]), int(vals[i]) + 10**9)
        assert got2.tolist() == [firsts[int(k)] for k in keys[:10].tolist()]


def test_erase_churn_compaction_reclaims_tombstones():
    import torch

    cap = 1 << 12
    idx = hasher.PrefixIndex(capacity=cap)
    rng = np.random.default_rng(9)
    live = {}
    for rnd in range(12):  # each round fills ~70% of the table, then erases it all
        keys = rng.integers(1, 2**62, int(0.7 * cap)).astype(np.uint64)
        idx.insert(keys, np.arange(len(keys), dtype=np.int64))  # compacts by itself when tombstones fill it
        live = {int(k): i for i, k in enumerate(keys.tolist())}
        if rnd < 11:
            idx.erase_device(torch.from_numpy(keys.view(np.int64)).cuda())
            torch.cuda.synchronize()
    assert idx.stats()[0] == len(live)
    ks = np.array(list(live), np.uint64)
    m, got = idx.lookup(np.arange(len(ks) + 1, dtype=np.int64), ks)
    assert np.all(m == 1) and got.tolist() == [live[int(k)] for k in ks.tolist()]
    # explicit compaction with nothing erased reclaims nothing; clear empties the table
    assert idx.compact() == 0
    idx.clear()
    assert idx.stats() == (0, 0)
    m, _ = idx.lookup(np.arange(len(ks) + 1, dtype=np.int64), ks)
    assert np.all(m == 0)
