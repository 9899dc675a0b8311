"""GPU parity: the CUDA path through the C ABI vs the pinned CPU oracle (bit-exact).

Runs on a B200 (`pytest -m gpu`).  Every comparison is against tests/golden (generated from the
compiled reference) or the oracle restatement pinned to it in test_oracle_pins.py.
"""
import ctypes as C

import numpy as np
import pytest
import torch

import pyoracle as po
from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

from paper_2603_21257_b200 import _capi  # noqa: E402
from paper_2603_21257_b200 import hasher, ingest  # noqa: E402
from paper_2603_21257_b200 import tiersim as t  # noqa: E402
from paper_2603_21257_b200.scorer import BatchScorer, DeviceQueue  # noqa: E402

CFGS = {"default": t.ClusterConfig(), "quad": t.ClusterConfig(compute_quadratic=1e-9, block_size_tokens=128)}


@pytest.fixture(scope="module")
def scorer():
    return BatchScorer(device=0)


def golden_queue(g, sl=slice(None)):
    return t.QueueArrays(**{k: np.array(g[k][sl]) for k, _ in t.QueueArrays.FIELDS})


# ---------------------------------------------------------------------------------------------
# K4 + K5: scorer and schedule order
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("cname", sorted(CFGS))
@pytest.mark.parametrize("policy", range(5))
def test_scores_and_order_bit_exact_vs_reference(golden, scorer, cname, policy):
    g = golden("ref_queue.npz")
    q = golden_queue(g)
    cfg = CFGS[cname]
    models = t.cost_models_from_config(cfg)
    assert np.array_equal(np.array([models.load.slope, models.load.intercept, models.comp.slope,
                                    models.comp.intercept]), g[f"{cname}_models"])
    tl, tc, pr, order = scorer.score(q, policy, models, cfg)
    assert np.array_equal(tl.view(np.uint64), g[f"{cname}_p{policy}_t_load"])
    assert np.array_equal(tc.view(np.uint64), g[f"{cname}_p{policy}_t_comp"])
    assert np.array_equal(pr.view(np.uint64), g[f"{cname}_p{policy}_primary"])
    assert np.array_equal(order, g[f"{cname}_p{policy}_order"])
    # device-resident variant
    out = scorer.score_device(DeviceQueue(q), policy, models, cfg)
    assert out["err_index"] == -1
    assert np.array_equal(out["primary"].cpu().numpy().view(np.uint64), g[f"{cname}_p{policy}_primary"])
    assert np.array_equal(out["order"].cpu().numpy(), g[f"{cname}_p{policy}_order"])


@pytest.mark.parametrize("policy", range(5))
def test_order_equals_reference_pick_next_drain(golden, scorer, policy):
    g = golden("ref_queue.npz")
    q = golden_queue(g, slice(0, 300))
    order = scorer.score(q, policy, t.cost_models_from_config(CFGS["default"]), CFGS["default"])[3]
    assert np.array_equal(order, g[f"drain300_p{policy}"])


def _req(i, arrival, deadline=None):
    return t.RequestSpec(id=i, arrival_time=arrival, context_tokens=1000, query_tokens=10, deadline=deadline)


def drain(queue, policy, costs):
    """test_scheduler.cpp:26-31 -- repeated pick_next, here backed by the GPU scorer."""
    queue = list(queue)
    out = []
    while (p := t.pick_next(queue, policy, costs, 0.0)) is not None:
        out.append(p.id)
    return out


def test_reference_scheduler_cases_on_gpu():
    """test_scheduler.cpp:42-89"""
    costs = {1: t.ServiceCost(0.361, 0.019), 2: t.ServiceCost(0.199, 0.025)}
    q = [_req(1, 0.0), _req(2, 0.0)]
    assert drain(q, t.PolicyKind.SjfCost, costs) == [2, 1]
    assert drain(q, t.PolicyKind.Fifo, costs) == [1, 2]
    a, b = _req(1, 0.0, 1.0), _req(2, 0.0, 0.8)
    costs = {1: t.ServiceCost(0.4, 0.1), 2: t.ServiceCost(0.05, 0.05)}
    assert drain([a, b], t.PolicyKind.Lstf, costs) == [1, 2]
    assert drain([a, b], t.PolicyKind.Edf, costs) == [2, 1]
    costs = {i: t.ServiceCost(0.1, 0.1) for i in (7, 9, 11)}
    assert drain([_req(7, 2.0), _req(9, 1.0)], t.PolicyKind.SjfCost, costs) == [9, 7]
    assert drain([_req(11, 1.0), _req(7, 1.0), _req(9, 1.0)], t.PolicyKind.SjfCost, costs) == [7, 9, 11]
    assert t.pick_next([], t.PolicyKind.Fifo, {}, 0.0) is None
    with pytest.raises(t.MissingDeadline, match="edf: request 1 has no deadline"):
        drain([_req(1, 0.0), _req(2, 0.0, 3.0)], t.PolicyKind.Edf, {})


def test_reference_scheduler_properties_on_gpu():
    """test_scheduler.cpp:104-183 properties through the GPU order (schedule_order = K4 + K5):
    scale invariance of SJF-cost, FIFO = arrival order, SJF-cost optimal for mean completion over
    every permutation (n <= 6), LSTF = EDF when every request costs the same."""
    import itertools

    rng = np.random.default_rng(11)
    for trial in range(20):
        n = int(rng.integers(2, 7))
        q = [t.RequestSpec(id=int(i) + 1, arrival_time=float(rng.integers(0, 3)), context_tokens=1000,
                           query_tokens=10, deadline=float(rng.random() * 5 + 1)) for i in range(n)]
        costs = {r.id: t.ServiceCost(float(rng.random()), float(rng.random())) for r in q}
        sjf = t.schedule_order(q, t.PolicyKind.SjfCost, costs)
        scaled = {k: t.ServiceCost(v.t_load * 8.0, v.t_comp * 8.0) for k, v in costs.items()}
        assert t.schedule_order(q, t.PolicyKind.SjfCost, scaled) == sjf  # scale invariance (x8 is exact)
        fifo = t.schedule_order(q, t.PolicyKind.Fifo, costs)
        assert fifo == [r.id for r in sorted(q, key=lambda r: (r.arrival_time, r.id))]
        total = {k: v.t_load + v.t_comp for k, v in costs.items()}
        def mean_completion(order):
            done, acc = 0.0, 0.0
            for i in order:
                done += total[i]
                acc += done
            return acc / n
        best = min(mean_completion(p) for p in itertools.permutations([r.id for r in q]))
        assert mean_completion(sjf) == pytest.approx(best, rel=1e-12)
        same = {r.id: t.ServiceCost(0.25, 0.125) for r in q}
        assert t.schedule_order(q, t.PolicyKind.Lstf, same) == t.schedule_order(q, t.PolicyKind.Edf, same)


def test_missing_deadline_reports_first_queue_index(golden, scorer):
    g = golden("ref_queue.npz")
    q = golden_queue(g)
    q.flags[[17, 40, 900]] &= np.uint8(0xFE)
    for pol in (t.PolicyKind.Edf, t.PolicyKind.Lstf):
        with pytest.raises(t.MissingDeadline, match=f"request {int(q.id[17])} has no deadline"):
            scorer.score(q, pol, t.cost_models_from_config(CFGS["default"]), CFGS["default"])
        out = None
        with pytest.raises(t.MissingDeadline):
            out = scorer.score_device(DeviceQueue(q), pol, t.cost_models_from_config(CFGS["default"]), CFGS["default"])
        assert out is None


def random_queue(n, seed):
    rng = np.random.default_rng(seed)
    q = t.QueueArrays(
        n,
        id=rng.permutation(n).astype(np.int64) * 3 - 7,
        arrival=np.round(rng.random(n) * 1000, 1),
        context_tokens=rng.integers(0, 200_000, n),
        query_tokens=rng.integers(1, 4000, n),
        cache_hit_ratio=rng.choice([0.0, 0.25, 0.5, 0.75, 0.9, 1.0, 0.3333333333333333], n),
        flags=np.where(rng.random(n) < 0.03, 3, 1).astype(np.uint8),
        deadline=np.round(rng.random(n) * 1000, 1) + 1000.0,
        measured_t_load=np.round(rng.random(n), 2),
        measured_t_comp=np.round(rng.random(n) * 0.1, 2),
    )
    q.arrival[100:2000] = 5.0  # heavy ties on arrival
    return q


@pytest.mark.parametrize("n", [1, 2, 2047, 2048, 2049, 4097, 100_000])
@pytest.mark.parametrize("policy", [t.PolicyKind.Fifo, t.PolicyKind.SjfPt, t.PolicyKind.Lstf])
def test_large_queue_matches_oracle(scorer, oracle, n, policy):
    q = random_queue(n, n)
    cfg = CFGS["default"]
    m = t.cost_models_from_config(cfg)
    tl, tc, pr, order = scorer.score(q, policy, m, cfg)
    st, err, otl, otc, opr = oracle.score_queue(q, int(policy), [m.load.slope, m.load.intercept, m.comp.slope,
                                                                 m.comp.intercept], cfg)
    assert st == 0
    assert np.array_equal(pr.view(np.uint64), opr.view(np.uint64))
    assert np.array_equal(tl.view(np.uint64), otl.view(np.uint64))
    assert np.array_equal(order, oracle.sort_order(opr, q.arrival, q.id))


@pytest.mark.parametrize("n", [1, 2, 3, 2049, 100_000])
@pytest.mark.parametrize("perturb", [None, "swap_last", "swap_first", "tie_ids"])
def test_presorted_queue_fast_path(scorer, oracle, n, perturb):
    """FIFO over an arrival-ordered queue is already in key order: K5 skips the merge sort
    (k_check_sorted / k_iota_if_sorted).  One displaced pair must fall back to the full sort."""
    q = random_queue(n, 7)
    order_in = np.lexsort((q.id, q.arrival))
    for name, _ in t.QueueArrays.FIELDS:
        setattr(q, name, getattr(q, name)[order_in].copy())
    if perturb == "swap_last" and n > 1:
        q.arrival[[-1, -2]] = q.arrival[[-2, -1]]
        q.id[[-1, -2]] = q.id[[-2, -1]]
    elif perturb == "swap_first" and n > 1:
        q.arrival[[0, 1]] = q.arrival[[1, 0]]
        q.id[[0, 1]] = q.id[[1, 0]]
    elif perturb == "tie_ids" and n > 2:
        q.arrival[:3] = q.arrival[0]  # equal arrival: ids decide
        q.id[:3] = q.id[:3][::-1].copy()
    cfg = CFGS["default"]
    m = t.cost_models_from_config(cfg)
    _, _, pr, order = scorer.score(q, t.PolicyKind.Fifo, m, cfg)
    want = oracle.sort_order(pr, q.arrival, q.id)
    assert np.array_equal(order, want)
    if perturb is None:
        assert np.array_equal(order, np.arange(n))


def test_signed_zero_and_infinite_keys_order(scorer, oracle):
    q = t.QueueArrays(4, id=np.array([4, 3, 2, 1]), arrival=np.array([0.0, -0.0, 0.0, 1.0]),
                      context_tokens=np.zeros(4, np.int64), query_tokens=np.ones(4, np.int64),
                      cache_hit_ratio=np.ones(4), flags=np.array([3, 3, 3, 3], np.uint8),
                      deadline=np.array([np.inf, 1.0, 1.0, np.inf]), measured_t_load=np.zeros(4),
                      measured_t_comp=np.array([0.0, 1.0, 1.0, 0.0]))
    for pol in range(5):
        _, _, pr, order = scorer.score(q, pol, t.CostModelPair(), t.ClusterConfig())
        assert np.array_equal(order, oracle.sort_order(pr, q.arrival, q.id)), pol


# ---------------------------------------------------------------------------------------------
# K3: prefix hasher
# ---------------------------------------------------------------------------------------------
def test_hash_frozen_vectors(golden):
    g = golden("hash_frozen.npz")
    assert np.array_equal(hasher.hash_prefix_chunks(g["offsets"], g["tokens"]), g["hashes"])


def test_hash_random_and_unaligned_vs_oracle(oracle):
    rng = np.random.default_rng(5)
    lens = rng.integers(0, 3000, 400)
    lens[:5] = [0, 255, 256, 257, 131072]
    offs = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=offs[1:])  # arbitrary (mostly unaligned) request starts
    doc = rng.integers(0, 7, len(lens))
    shared = rng.integers(0, 3000, len(lens))
    toks = oracle.gen_tokens(99, offs, doc, shared)
    assert np.array_equal(hasher.hash_prefix_chunks(offs, toks), oracle.hash_prefix_chunks(offs, toks))


def test_hash_device_path_and_token_generator(oracle):
    rng = np.random.default_rng(6)
    lens = (rng.integers(1, 600, 1000) * 4).astype(np.int64)
    offs = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=offs[1:])
    doc = rng.integers(0, 16, len(lens)).astype(np.int64)
    shared = rng.integers(0, 2000, len(lens)).astype(np.int64)
    dev = torch.device("cuda", 0)
    d_offs, d_doc, d_sh = (torch.from_numpy(x).to(dev) for x in (offs, doc, shared))
    d_tok = torch.empty(int(offs[-1]), dtype=torch.int32, device=dev)
    hasher.gen_tokens_device(3, d_offs, d_doc, d_sh, d_tok)
    want_tok = oracle.gen_tokens(3, offs, doc, shared)
    assert np.array_equal(d_tok.cpu().numpy(), want_tok)
    coff = hasher.chunk_offsets(offs)
    d_out = torch.empty(int(coff[-1]), dtype=torch.int64, device=dev)
    hasher.hash_prefix_chunks_device(d_offs, d_tok, torch.from_numpy(coff).to(dev), d_out)
    torch.cuda.synchronize()
    assert np.array_equal(d_out.cpu().numpy().view(np.uint64), oracle.hash_prefix_chunks(offs, want_tok))


# ---------------------------------------------------------------------------------------------
# K1 / K1b / CE+K2: L2 -> L1 ingest through the paged allocator
# ---------------------------------------------------------------------------------------------
SMALL = ingest.KVShape(layers=4, kv_heads=8, head_dim=128, chunk_tokens=256, page_tokens=16)


def build_scenario(shape, n_slots=8, num_pages=200, seed=17, pool=None):
    """Pool of synthetic chunks; three requests through the L1 ledger (one deferred, then granted
    after a release) so the block table is a non-trivial permutation of pages.  `pool`: use this
    (already filled) pool instead of a fresh host pool."""
    if pool is None:
        pool = ingest.ChunkPool(shape, n_slots)
        pool.fill_synthetic(seed)
    n_slots = pool.n_slots
    arena = torch.zeros(shape.layers * 2 * num_pages * shape.page_tokens * shape.heads_local * shape.head_dim * 2,
                        dtype=torch.uint8, device="cuda")
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=4, max_chunks=12, arena=arena)
    cb = shape.page_bytes * shape.pages_per_chunk
    items = []
    # request 10: 6 chunks; request 11: 5 chunks; release 10; request 12: 7 chunks (partly deferred)
    for c in range(6):
        assert l1.request(10, c, cb)[0]
    for c in range(5):
        g, row11 = l1.request(11, c, cb)
        assert g
    granted_12 = []
    for c in range(7):
        g, row12 = l1.request(12, c, cb)
        if g:
            granted_12.append(c)
    assert l1.deferred_count() > 0  # 18 chunks x 16 pages > 200 pages
    grants = l1.release_request(10)
    granted_12 += [b for (rid, b, row, nb) in grants if rid == 12]
    assert l1.deferred_count() == 0 and sorted(granted_12) == list(range(7))
    rng = np.random.default_rng(seed)
    for c in range(5):
        items.append((int(rng.integers(n_slots)), row11, c))
    for c in range(7):
        items.append((int(rng.integers(n_slots)), row12, c))
    l1.sync_block_table()
    return pool, l1, ingest.items_numpy(*zip(*items))


def alloc_ref_block_table(shape, num_pages):
    """alloc_ref (orc_pages FIFO free list) driven by the same ledger decisions as build_scenario."""
    lib = po.restate()
    pages = lib.orc_pages_new(num_pages)
    ppc = shape.pages_per_chunk
    rows = {}
    buf = (C.c_int32 * ppc)()
    def take(rid, c):
        assert lib.orc_pages_take(pages, ppc, buf) == ppc
        rows.setdefault(rid, {})[c] = list(buf)
    for c in range(6):
        take(10, c)
    for c in range(5):
        take(11, c)
    pending = []
    for c in range(7):
        if lib.orc_pages_available(pages) >= ppc and not pending:
            take(12, c)
        else:
            pending.append(c)
    rows10 = rows.pop(10)
    freed = [p for c in range(6) for p in rows10[c]]
    arr = (C.c_int32 * len(freed))(*freed)
    lib.orc_pages_give(pages, len(freed), arr)
    for c in pending:
        take(12, c)
    lib.orc_pages_free(pages)
    return rows


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_allocator_random_script_matches_ledger_and_alloc_ref(seed):
    """Random request/release scripts: grant/defer decisions, FIFO grant lists, reserved bytes
    and page ids of the L1 allocator equal TierLedger (restated, pinned to the reference) driving
    the FIFO page free list (alloc_ref)."""
    lib = po.restate()
    rng = np.random.default_rng(seed)
    shape = SMALL
    num_pages = 16 * 20
    pb = shape.page_bytes * shape.pages_per_chunk  # one chunk reservation
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=64, max_chunks=8)
    led = lib.orc_ledger_new(num_pages * shape.page_bytes)
    pages = lib.orc_pages_new(num_pages)
    held = {}   # request -> list of its pages in grant order (alloc_ref)
    waiting = {}
    live = []
    buf = (C.c_int32 * 16)()
    for step in range(300):
        if live and (rng.random() < 0.35 or len(live) >= 48):  # 64 block-table rows
            rid = live.pop(int(rng.integers(len(live))))
            if waiting.get(rid):
                live.append(rid)
                continue
            got = l1.release_request(rid)
            freed = held.pop(rid)
            arr = (C.c_int32 * len(freed))(*freed)
            lib.orc_pages_give(pages, len(freed), arr)
            rid_o, blk_o, by_o, n = (C.c_int64 * 64)(), (C.c_int32 * 64)(), (C.c_int64 * 64)(), C.c_int64()
            assert lib.orc_ledger_release(led, len(freed) * shape.page_bytes, rid_o, blk_o, by_o, 64, C.byref(n)) == 0
            want = [(rid_o[i], blk_o[i]) for i in range(n.value)]
            assert [(g[0], g[1]) for g in got] == want
            for r_, b_ in want:
                assert lib.orc_pages_take(pages, 16, buf) == 16
                held.setdefault(r_, []).extend(list(buf))
                waiting[r_] -= 1
                bt = l1.block_table()[[g[2] for g in got if g[0] == r_][0], b_ * 16:(b_ + 1) * 16]
                assert list(bt) == list(buf)
        else:
            rid = 1000 + step
            nch = int(rng.integers(1, 5))
            for c in range(nch):
                g, row = l1.request(rid, c, pb)
                gr = C.c_int()
                assert lib.orc_ledger_request(led, rid, c, pb, C.byref(gr)) == 0
                assert bool(gr.value) == g
                if g:
                    assert lib.orc_pages_take(pages, 16, buf) == 16
                    held.setdefault(rid, []).extend(list(buf))
                    assert list(l1.block_table()[row, c * 16:(c + 1) * 16]) == list(buf)
                else:
                    waiting[rid] = waiting.get(rid, 0) + 1
                    held.setdefault(rid, [])
            live.append(rid)
        assert l1.reserved() == lib.orc_ledger_reserved(led)
        assert l1.deferred_count() == lib.orc_ledger_deferred(led)
    lib.orc_ledger_free(led)
    lib.orc_pages_free(pages)


def test_page_ids_match_alloc_ref():
    pool, l1, items = build_scenario(SMALL)
    bt = l1.block_table()
    want = alloc_ref_block_table(SMALL, l1.num_pages)
    rows = {11: items["bt_row"][0], 12: items["bt_row"][-1]}
    for rid, chunks in want.items():
        for c, pages in chunks.items():
            assert list(bt[rows[rid], c * 16:(c + 1) * 16]) == pages


@pytest.mark.parametrize("mode", ["zerocopy", "bulk", "ce", "auto"])
def test_ingest_bit_exact_vs_scatter_ref(oracle, mode):
    pool, l1, items = build_scenario(SMALL)
    ingest.ingest(l1, pool, items, mode=ingest.MODES[mode])
    torch.cuda.synchronize()
    got = l1.arena.cpu().numpy()
    want = oracle.scatter_ref(SMALL, pool.slot_view(0, pool.n_slots), items, l1.block_table(), l1.num_pages)
    assert np.array_equal(got, want)
    assert ingest.verify_synthetic(l1, pool, items, seed=17) == 0


def test_k2_scatter_alone_bit_exact(oracle):
    """tsb_scatter_device: K2 from an HBM staging buffer holding layers [1, 3) of each item."""
    pool, l1, items = build_scenario(SMALL)
    lo, hi = 1, 3
    chunks = pool.slot_view(0, pool.n_slots).reshape(pool.n_slots, SMALL.layers, -1)
    staging = torch.from_numpy(np.ascontiguousarray(chunks[items["src_slot"], lo:hi]).reshape(-1)).cuda()
    dev_items = torch.from_numpy(items.view(np.uint8).copy()).cuda()
    t.check(_capi.lib.tsb_scatter_device(l1.handle, staging.data_ptr(), dev_items.data_ptr(), len(items), lo, hi,
                                         torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = oracle.scatter_ref(SMALL, pool.slot_view(0, pool.n_slots), items, l1.block_table(), l1.num_pages, lo, hi)
    assert np.array_equal(l1.arena.cpu().numpy(), want)


@pytest.mark.parametrize("tp", [(1, 0), (4, 1)])
def test_k2_scatter_packed_bit_exact(oracle, tp):
    """tsb_scatter_device_packed: K2 from the CE path's staging format (this rank's heads only,
    layers [1, 3) of each item packed)."""
    shape = SMALL.with_rank(*tp)
    pool, l1, items = build_scenario(shape)
    lo, hi = 1, 3
    hl, h0 = shape.heads_local, shape.tp_rank * shape.heads_local
    chunks = pool.slot_view(0, pool.n_slots).view(np.uint16).reshape(pool.n_slots, SMALL.layers, 2, 256, 8, 128)
    packed = np.ascontiguousarray(chunks[items["src_slot"], lo:hi, :, :, h0:h0 + hl, :])
    staging = torch.from_numpy(packed.view(np.uint8).reshape(-1)).cuda()
    dev_items = torch.from_numpy(items.view(np.uint8).copy()).cuda()
    t.check(_capi.lib.tsb_scatter_device_packed(l1.handle, staging.data_ptr(), dev_items.data_ptr(), len(items), lo,
                                                hi, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = oracle.scatter_ref(shape, pool.slot_view(0, pool.n_slots), items, l1.block_table(), l1.num_pages, lo, hi)
    assert np.array_equal(l1.arena.cpu().numpy(), want)


@pytest.mark.parametrize("variant", [0, 1])
def test_ingest_ce_copy_variants_bit_exact(oracle, variant):
    """CE strategies: per-item memcpy, 2D copy per run of consecutive slots."""
    pool, l1, items = build_scenario(SMALL)
    items["src_slot"] = (np.arange(len(items)) + 2) % pool.n_slots  # runs 2..7, 0..5
    ingest.set_ce(variant)
    try:
        ingest.ingest(l1, pool, items, mode=ingest.CE)
        ingest.ingest(l1, pool, items[::-1].copy(), 1, 3, mode=ingest.CE)
        torch.cuda.synchronize()
    finally:
        ingest.set_ce()
    want = oracle.scatter_ref(SMALL, pool.slot_view(0, pool.n_slots), items, l1.block_table(), l1.num_pages)
    assert np.array_equal(l1.arena.cpu().numpy(), want)


@pytest.mark.parametrize("tp", [(2, 0), (2, 1), (4, 3), (8, 5)])
@pytest.mark.parametrize("mode", ["zerocopy", "bulk", "ce", "ce_runs"])
def test_ingest_head_sharded_bit_exact(oracle, tp, mode):
    """Head-sharded slices; "ce" = strided 3D copies of random slots (runs of 1), "ce_runs" =
    consecutive slots 2..7, 0..5 (multi-slot 3D copies), both then K2 over the packed staging."""
    shape = SMALL.with_rank(*tp)
    pool, l1, items = build_scenario(shape)
    if mode == "ce_runs":
        items["src_slot"] = (np.arange(len(items)) + 2) % pool.n_slots
        mode = "ce"
    ingest.ingest(l1, pool, items, mode=ingest.MODES[mode])
    torch.cuda.synchronize()
    want = oracle.scatter_ref(shape, pool.slot_view(0, pool.n_slots), items, l1.block_table(), l1.num_pages)
    assert np.array_equal(l1.arena.cpu().numpy(), want)


def test_ingest_per_layer_with_events_equals_whole(oracle):
    pool, l1, items = build_scenario(SMALL)
    s = torch.cuda.Stream()
    want = oracle.scatter_ref(SMALL, pool.slot_view(0, pool.n_slots), items, l1.block_table(), l1.num_pages)
    for mode in (ingest.BULK, ingest.ZEROCOPY, ingest.CE):
        l1.arena.zero_()
        torch.cuda.synchronize()
        evs = [torch.cuda.Event() for _ in range(SMALL.layers)]
        with torch.cuda.stream(s):
            ingest.ingest(l1, pool, items, 0, 2, mode=mode, stream=s, layer_events=evs[:2])
            for layer in range(2, SMALL.layers):
                ingest.ingest(l1, pool, items, layer, layer + 1, mode=mode, stream=s, layer_events=[evs[layer]])
        for layer, e in enumerate(evs):
            e.synchronize()
            page0 = l1.block_table()[items["bt_row"][0], items["chunk_index"][0] * 16]
            assert l1.layer(layer, torch.int16)[0, page0].abs().sum().item() > 0
        evs[-1].synchronize()
        assert np.array_equal(l1.arena.cpu().numpy(), want), mode
    # vLLM flash-attn view: [2, num_pages, page_tokens, heads, head_dim]
    assert tuple(l1.layer(0).shape) == (2, 200, 16, 8, 128)


@pytest.mark.parametrize("mode", ["zerocopy", "bulk", "ce"])
def test_ingest_sparse_layer_events(oracle, mode):
    """Fences on some layers only: the SM kernels launch once per span of layers ending at a
    fence (here [0,1) and [1,4)); each fence still means "layers up to here are resident"."""
    pool, l1, items = build_scenario(SMALL)
    s = torch.cuda.Stream()
    e0, e3 = torch.cuda.Event(), torch.cuda.Event()
    launches = _capi.lib.tsb_kernel_launch_count()
    with torch.cuda.stream(s):
        ingest.ingest(l1, pool, items, 0, SMALL.layers, mode=ingest.MODES[mode], stream=s,
                      layer_events=[e0, None, None, e3])
    e0.synchronize()
    page0 = l1.block_table()[items["bt_row"][0], items["chunk_index"][0] * 16]
    assert l1.layer(0, torch.int16)[0, page0].abs().sum().item() > 0
    e3.synchronize()
    if mode != "ce":
        assert _capi.lib.tsb_kernel_launch_count() - launches == 2
    want = oracle.scatter_ref(SMALL, pool.slot_view(0, pool.n_slots), items, l1.block_table(), l1.num_pages)
    assert np.array_equal(l1.arena.cpu().numpy(), want)


@pytest.mark.parametrize("fences", ["every", "sparse", "none"])
@pytest.mark.parametrize("layout", ["flash_attn", "flashinfer_nhd", "flashinfer_hnd"])
@pytest.mark.parametrize("tp", [(1, 0), (2, 1)])
def test_ce_direct_bit_exact(oracle, layout, tp, fences):
    """CE-direct: the copy engines write the pages (one 3D copy per run of consecutive pages over
    K|V x the layers up to the next fence), no kernel launched; flash-attn / NHD pages of
    full-head chunks, else UNSUPPORTED."""
    lay = ingest.LAYOUTS[layout]
    shape = SMALL.with_rank(*tp)
    pool = ingest.ChunkPool(SMALL, 8)
    pool.fill_synthetic(29)
    num_pages = 200
    arena = torch.zeros(shape.layers * 2 * num_pages * 16 * shape.heads_local * 128 * 2, dtype=torch.uint8,
                        device="cuda")
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=2, max_chunks=12, arena=arena, layout=lay)
    rows = [l1.request(5, c, shape.page_bytes * 16)[1] for c in range(7)]
    bt = l1.block_table()
    bt[rows[0], 16:48] = bt[rows[0], 16:48][::-1].copy()  # chunks 1-2: pages in reverse (no merging)
    l1.sync_block_table()
    items = ingest.items_numpy([3, 4, 5, 6, 0, 1, 7], rows, range(7))
    supported = tp[0] == 1 and layout != "flashinfer_hnd"
    assert bool(_capi.lib.tsb_ingest_ce_direct_supported(l1.handle, pool.handle)) == supported
    if not supported:
        with pytest.raises(t.Unsupported):
            ingest.ingest(l1, pool, items, mode=ingest.CE_DIRECT)
        return
    evs = None
    if fences == "every":
        evs = [torch.cuda.Event() for _ in range(shape.layers)]
    elif fences == "sparse":  # spans of 1 and of several layers
        evs = [torch.cuda.Event() if l in (0, shape.layers - 1) else None for l in range(shape.layers)]
    launches = _capi.lib.tsb_kernel_launch_count()
    ingest.ingest(l1, pool, items, mode=ingest.CE_DIRECT, layer_events=evs)
    if evs:
        evs[0].synchronize()
    torch.cuda.synchronize()
    assert _capi.lib.tsb_kernel_launch_count() == launches  # no SM work
    want = oracle.scatter_ref(shape, pool.slot_view(0, 8), items, l1.block_table(), num_pages, layout=lay)
    assert np.array_equal(arena.cpu().numpy(), want)


@pytest.mark.parametrize("layout", ["flashinfer_nhd", "flashinfer_hnd"])
@pytest.mark.parametrize("mode", ["zerocopy", "bulk", "ce", "auto"])
@pytest.mark.parametrize("tp", [(1, 0), (2, 1), (8, 6)])
def test_ingest_layouts_bit_exact(oracle, layout, mode, tp):
    """The consumer's page layout (vLLM FlashInfer NHD / HND): same pages, permuted addresses."""
    lay = ingest.LAYOUTS[layout]
    shape = SMALL.with_rank(*tp)
    pool = ingest.ChunkPool(SMALL, 8)
    pool.fill_synthetic(17)
    num_pages = 200
    arena = torch.zeros(shape.layers * 2 * num_pages * 16 * shape.heads_local * 128 * 2, dtype=torch.uint8,
                        device="cuda")
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=2, max_chunks=12, arena=arena, layout=lay)
    rows = [l1.request(5, c, shape.page_bytes * 16)[1] for c in range(7)]
    l1.sync_block_table()
    items = ingest.items_numpy([3, 4, 5, 6, 0, 1, 7], rows, range(7))
    ingest.ingest(l1, pool, items, mode=ingest.MODES[mode])
    torch.cuda.synchronize()
    want = oracle.scatter_ref(shape, pool.slot_view(0, 8), items, l1.block_table(), num_pages, layout=lay)
    assert np.array_equal(arena.cpu().numpy(), want)
    assert ingest.verify_synthetic(l1, pool, items, seed=17) == 0
    assert tuple(l1.layer(0).shape)[:2] == (num_pages, 2)


@pytest.mark.parametrize("layout", ["flash_attn", "flashinfer_nhd", "flashinfer_hnd"])
@pytest.mark.parametrize("tp", [(1, 0), (2, 1), (8, 6)])
@pytest.mark.parametrize("source", ["host", "device"])
def test_k1b_tensor_map_tma_bit_exact(oracle, layout, tp, source):
    """K1b: one tensor-map TMA load per page segment (2D map for NHD, 3D (D, rows, heads) map for HND
    pages -- the TMA unit does the per-head transpose), from a host or an HBM pool, and as K2 from
    the CE staging ring (tsb_ingest_set_scatter(1)): bit-exact against scatter_ref."""
    lay = ingest.LAYOUTS[layout]
    shape = SMALL.with_rank(*tp)
    pool = ingest.ChunkPool(SMALL, 8) if source == "host" else ingest.ChunkPool.create_device(SMALL, 8)
    pool.fill_synthetic(23)
    host = ingest.ChunkPool(SMALL, 8)
    host.fill_synthetic(23)
    num_pages = 200
    arena = torch.zeros(shape.layers * 2 * num_pages * 16 * shape.heads_local * 128 * 2, dtype=torch.uint8,
                        device="cuda")
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=2, max_chunks=12, arena=arena, layout=lay)
    rows = [l1.request(5, c, shape.page_bytes * 16)[1] for c in range(7)]
    l1.sync_block_table()
    items = ingest.items_numpy([3, 4, 5, 6, 0, 1, 7], rows, range(7))
    want = oracle.scatter_ref(shape, host.slot_view(0, 8), items, l1.block_table(), num_pages, layout=lay)
    ingest.ingest(l1, pool, items, mode=ingest.BULK)
    torch.cuda.synchronize()
    assert np.array_equal(arena.cpu().numpy(), want)
    if source == "host":  # K2 on the TMA kernel, over the packed CE staging ring
        arena.zero_()
        t.check(_capi.lib.tsb_ingest_set_scatter(1, 0))
        try:
            ingest.ingest(l1, pool, items, mode=ingest.CE)
            torch.cuda.synchronize()
        finally:
            t.check(_capi.lib.tsb_ingest_set_scatter(0, 0))
        assert np.array_equal(arena.cpu().numpy(), want)


def test_layout_fixed_once_reserved():
    l1 = ingest.PagedKVCache(SMALL, 64, max_rows=1, max_chunks=2)
    l1.request(1, 0, SMALL.page_bytes * 16)
    with pytest.raises(t.ValidationError):
        t.check(_capi.lib.tsb_l1_set_layout(l1.handle, ingest.LAYOUT_FLASHINFER_NHD))
    l1.release_request(1)
    t.check(_capi.lib.tsb_l1_set_layout(l1.handle, ingest.LAYOUT_FLASHINFER_HND))
    assert _capi.lib.tsb_l1_layout(l1.handle) == ingest.LAYOUT_FLASHINFER_HND


@pytest.mark.parametrize("tp", [(1, 0), (4, 2)])
def test_ce_layer_groups_with_subranges_and_fences(oracle, tp):
    """CE groups consecutive layers up to the next fence: a layer sub-range [1, 4) with a fence only
    on its last layer (one group), then layer 0 alone with its own fence; runs of consecutive
    slots and scattered slots mixed.  Equals the whole scatter."""
    shape = SMALL.with_rank(*tp)
    pool = ingest.ChunkPool(SMALL, 8)
    pool.fill_synthetic(23)
    num_pages = 200
    arena = torch.zeros(shape.layers * 2 * num_pages * 16 * shape.heads_local * 128 * 2, dtype=torch.uint8,
                        device="cuda")
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=2, max_chunks=12, arena=arena)
    rows = [l1.request(9, c, shape.page_bytes * 16)[1] for c in range(8)]
    l1.sync_block_table()
    items = ingest.items_numpy([2, 3, 4, 5, 7, 0, 1, 6], rows, range(8))
    e_last, e0 = torch.cuda.Event(), torch.cuda.Event()
    ingest.ingest(l1, pool, items, 1, 4, mode=ingest.CE, layer_events=[None, None, e_last])
    ingest.ingest(l1, pool, items, 0, 1, mode=ingest.CE, layer_events=[e0])
    e0.synchronize()
    e_last.synchronize()
    want = oracle.scatter_ref(shape, pool.slot_view(0, 8), items, l1.block_table(), num_pages)
    assert np.array_equal(arena.cpu().numpy(), want)


@pytest.mark.parametrize("tp", [(1, 0), (4, 1)])
def test_ce_group_cap_bit_exact(oracle, tp):
    """A per-L1 CE group cap of 3 item-layers (what the stage applies, at 128 MiB, while a prefill
    runs): groups of 3 items per layer inside the 1 GiB ring, with per-layer fences."""
    shape = SMALL.with_rank(*tp)
    lb = 2 * shape.chunk_tokens * shape.heads_local * shape.head_dim * shape.dtype_bytes
    pool, l1, items = build_scenario(shape)
    assert l1.ce_group_bytes == 0
    l1.ce_group_bytes = 3 * lb
    assert l1.ce_group_bytes == 3 * lb
    evs = [torch.cuda.Event() for _ in range(shape.layers)]
    ingest.ingest(l1, pool, items, mode=ingest.CE, layer_events=evs)
    torch.cuda.synchronize()
    with pytest.raises(t.ValidationError):
        l1.ce_group_bytes = -1
    l1.ce_group_bytes = 0
    want = oracle.scatter_ref(shape, pool.slot_view(0, pool.n_slots), items, l1.block_table(), l1.num_pages)
    assert np.array_equal(l1.arena.cpu().numpy(), want)


@pytest.mark.parametrize("tp", [(1, 0), (4, 1)])
def test_ce_small_staging_splits_items(oracle, tp):
    """A staging half that holds 3 item-layers: CE splits the items of each layer into groups of 3
    (no layer grouping), ping-ponging the two halves many times per call."""
    shape = SMALL.with_rank(*tp)
    lb = 2 * shape.chunk_tokens * shape.heads_local * shape.head_dim * shape.dtype_bytes
    pool, l1, items = build_scenario(shape)
    ingest.set_ce(1, 2 * 3 * lb)
    try:
        ingest.ingest(l1, pool, items, mode=ingest.CE)
        torch.cuda.synchronize()
    finally:
        ingest.set_ce()
    want = oracle.scatter_ref(shape, pool.slot_view(0, pool.n_slots), items, l1.block_table(), l1.num_pages)
    assert np.array_equal(l1.arena.cpu().numpy(), want)


def test_auto_mode_resolution():
    """AUTO: host pool + full heads -> CE; head-sharded -> CE when consecutive-slot runs carry
    >= 3.1 MB per strided copy, else K1; device pool or device items -> K1 (zero-copy kernel)."""
    shape = ingest.LLAMA3_70B.with_rank(8, 3)  # 256 B runs; one chunk's layer slice = 128 KiB
    pool = ingest.ChunkPool(ingest.LLAMA3_70B, 40)
    l1 = ingest.PagedKVCache(shape, 64, max_rows=1, max_chunks=40)
    run = ingest.items_numpy(np.arange(40), np.zeros(40, np.int32), np.arange(40))   # 40 x 128 KiB = 5.2 MB
    short = ingest.items_numpy(np.arange(20), np.zeros(20, np.int32), np.arange(20))  # 2.6 MB per copy
    scattered = run.copy()
    scattered["src_slot"] = np.random.default_rng(0).permutation(40)
    assert ingest.resolve_mode(l1, pool, run) == ingest.CE
    assert ingest.resolve_mode(l1, pool, short) == ingest.ZEROCOPY
    assert ingest.resolve_mode(l1, pool, scattered) == ingest.ZEROCOPY
    assert ingest.resolve_mode(l1, pool, None) == ingest.ZEROCOPY
    assert ingest.resolve_mode(l1, pool, scattered, ingest.BULK) == ingest.BULK
    full = ingest.PagedKVCache(ingest.LLAMA3_70B, 64, max_rows=1, max_chunks=40)
    assert ingest.resolve_mode(full, pool, scattered) == ingest.CE
    dpool = ingest.ChunkPool.create_device(ingest.LLAMA3_70B, 2)
    assert ingest.resolve_mode(full, dpool, run[:1]) == ingest.ZEROCOPY
    with pytest.raises(t.ValidationError):
        ingest.resolve_mode(full, pool, run, 7)


def test_ingest_errors_fail_loudly():
    pool, l1, items = build_scenario(SMALL)
    with pytest.raises(t.ValidationError):
        ingest.ingest(l1, pool, items, 3, 3)
    with pytest.raises(t.Unsupported):  # the copy engines read host pools only
        dpool = ingest.ChunkPool.create_device(SMALL, 2)
        it0 = items[:1].copy()
        it0["src_slot"] = 0
        ingest.ingest(l1, dpool, it0, mode=ingest.CE)
    with pytest.raises(t.CapacityError):
        l1.request(99, 0, 10**15)
    with pytest.raises(t.ValidationError):
        l1.request(99, 0, 12345)  # not a whole number of pages
    with pytest.raises(t.ValidationError):
        l1.release_request(4242)


@pytest.mark.parametrize("mode", ["bulk", "ce"])
def test_config1_full_size_llama8b_32k(mode):
    """configs[0]: Llama-3.1-8B KV, one 32K prefix = 128 chunks (4.29 GB) -> 2048 pages, per layer.
    Size-independent checks: every byte of every page equals the synthetic word of the source
    position it must come from (verify kernel), plus sampled segments compared on the host."""
    shape = ingest.LLAMA31_8B
    pool = ingest.ChunkPool(shape, 128)
    pool.fill_synthetic(5)
    l1 = ingest.PagedKVCache(shape, 2048, max_rows=1, max_chunks=128)
    cb = shape.page_bytes * 16
    rows = []
    for c in range(128):
        g, row = l1.request(1, c, cb)
        assert g
    assert l1.free_pages() == 0
    items = ingest.items_numpy(np.random.default_rng(1).permutation(128), [row] * 128, np.arange(128))
    l1.sync_block_table()
    for layer in range(shape.layers):
        ingest.ingest(l1, pool, items, layer, layer + 1, mode=ingest.MODES[mode])
    torch.cuda.synchronize()
    assert ingest.verify_synthetic(l1, pool, items, seed=5) == 0
    bt = l1.block_table()
    rng = np.random.default_rng(2)
    poolv = pool.slot_view(0, 128).view(np.uint16).reshape(128, 32, 2, 256, 8, 128)
    for _ in range(64):
        i, layer, kv, j = rng.integers(128), rng.integers(32), rng.integers(2), rng.integers(16)
        page = bt[row, items["chunk_index"][i] * 16 + j]
        got = l1.layer(layer, torch.int16)[kv, page].cpu().numpy().view(np.uint16)
        want = poolv[items["src_slot"][i], layer, kv, j * 16:(j + 1) * 16]
        assert np.array_equal(got, want)
    assert l1.release_request(1) == [] and l1.free_pages() == 2048


@pytest.mark.parametrize("tp", [2, 8])
def test_config2_full_size_llama70b_head_shards(tp):
    """configs[2]: Llama-3-70B KV, one 32K prefix (128 chunks of 80 MiB), rank tp-1 of a tp-way
    head split, AUTO (strided copy-engine 3D copies + K2), per-layer fences.  Every word of every
    page is checked against the synthetic source (verify kernel)."""
    full = ingest.LLAMA3_70B
    shape = full.with_rank(tp, tp - 1)
    pool = ingest.ChunkPool(full, 128)
    pool.fill_synthetic(11)
    l1 = ingest.PagedKVCache(shape, 2048, max_rows=1, max_chunks=128)
    for c in range(128):
        g, row = l1.request(1, c, shape.page_bytes * 16)
        assert g
    l1.sync_block_table()
    items = ingest.items_numpy(np.arange(128), [row] * 128, np.arange(128))
    assert ingest.resolve_mode(l1, pool, items) == ingest.CE
    evs = [torch.cuda.Event() for _ in range(shape.layers)]
    ingest.ingest(l1, pool, items, layer_events=evs)
    evs[-1].synchronize()
    assert ingest.verify_synthetic(l1, pool, items, seed=11) == 0


# ---------------------------------------------------------------------------------------------
# Geometry generality and edge cases
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("geom", [
    dict(layers=3, kv_heads=4, head_dim=64, dtype_bytes=2, chunk_tokens=128, page_tokens=16),
    dict(layers=2, kv_heads=8, head_dim=256, dtype_bytes=1, chunk_tokens=256, page_tokens=32),   # fp8 KV
    dict(layers=2, kv_heads=2, head_dim=128, dtype_bytes=2, chunk_tokens=64, page_tokens=8),
    dict(layers=1, kv_heads=16, head_dim=128, dtype_bytes=2, chunk_tokens=256, page_tokens=16),
])
@pytest.mark.parametrize("mode", ["zerocopy", "bulk", "ce"])
def test_ingest_geometries_bit_exact(oracle, geom, mode):
    shape = ingest.KVShape(**geom)
    ppc = shape.pages_per_chunk
    pool = ingest.ChunkPool(shape, 6)
    pool.fill_synthetic(29)
    num_pages = 8 * ppc + 3
    arena = torch.zeros(shape.layers * 2 * num_pages * shape.page_tokens * shape.heads_local * shape.head_dim *
                        shape.dtype_bytes, dtype=torch.uint8, device="cuda")
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=2, max_chunks=8, arena=arena)
    cb = shape.page_bytes * ppc
    items = []
    for c in range(5):
        g, row = l1.request(7, c, cb)
        assert g
        items.append(((c * 3) % 6, row, c))
    l1.sync_block_table()
    it = ingest.items_numpy(*zip(*items))
    try:
        ingest.ingest(l1, pool, it, mode=ingest.MODES[mode])
    except t.Unsupported:
        pytest.skip("segment too large for the bulk ring")
    torch.cuda.synchronize()
    want = oracle.scatter_ref(shape, pool.slot_view(0, 6), it, l1.block_table(), num_pages)
    assert np.array_equal(l1.arena.cpu().numpy(), want)


def test_ingest_empty_and_bounds():
    pool, l1, items = build_scenario(SMALL)
    ingest.ingest(l1, pool, items[:0])  # no items: no work, no error
    evs = [torch.cuda.Event() for _ in range(SMALL.layers)]
    ingest.ingest(l1, pool, items[:0], layer_events=evs)
    for e in evs:
        e.synchronize()  # fences still recorded
    with pytest.raises(t.ValidationError):
        ingest.ingest(l1, pool, items, 0, SMALL.layers + 1)
    with pytest.raises(t.ValidationError):
        l1.request(55, 12, SMALL.page_bytes * 16)  # chunk index beyond the block-table row
    for field, bad in (("src_slot", pool.n_slots), ("src_slot", -1), ("bt_row", 4), ("chunk_index", 12)):
        it = items[:2].copy()
        it[field][1] = bad
        with pytest.raises(t.ValidationError, match="outside the pool"):
            ingest.ingest(l1, pool, it)
    ingest.ingest(l1, pool, items)  # the context is still healthy
    torch.cuda.synchronize()


def test_hash_edge_lengths(oracle):
    offs = np.array([0, 0, 1, 255, 511, 767, 768 + 1_000_000], np.int64)  # lengths 0,1,254,256,256,1_000_001
    doc = np.zeros(len(offs) - 1, np.int64)
    toks = oracle.gen_tokens(5, offs, doc, np.diff(offs))
    got = hasher.hash_prefix_chunks(offs, toks)
    assert np.array_equal(got, oracle.hash_prefix_chunks(offs, toks))
    assert len(got) == sum(int(x) // 256 for x in np.diff(offs))


@pytest.mark.parametrize("policy", [t.PolicyKind.SjfCost, t.PolicyKind.Edf])
def test_scorer_one_million_requests(scorer, oracle, policy):
    q = random_queue(1_000_000, 11)
    cfg = CFGS["quad"]
    m = t.cost_models_from_config(cfg)
    tl, tc, pr, order = scorer.score(q, policy, m, cfg)
    st, err, otl, otc, opr = oracle.score_queue(q, int(policy), [m.load.slope, m.load.intercept, m.comp.slope,
                                                                 m.comp.intercept], cfg)
    assert np.array_equal(pr.view(np.uint64), opr.view(np.uint64))
    assert np.array_equal(order, oracle.sort_order(opr, q.arrival, q.id))


def test_scorer_empty_queue(scorer):
    q = t.QueueArrays(0)
    tl, tc, pr, order = scorer.score(q, t.PolicyKind.Fifo, t.CostModelPair(), t.ClusterConfig())
    assert len(order) == 0


def test_hash_aligned_layout_and_phase1(oracle):
    """K3 on a layout with 16-byte-aligned request starts (gaps between requests) gives the same
    chained hashes as the packed layout; phase 1 alone gives unchained per-chunk digests."""
    rng = np.random.default_rng(12)
    n = 300
    lens = rng.integers(0, 3000, n)
    lens[::7] = rng.integers(250, 260, len(lens[::7]))  # around one chunk
    doc = rng.integers(0, 20, n)
    shared = lens // 2
    packed = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=packed[1:])
    toks = oracle.gen_tokens(5, packed, doc, shared)
    want = oracle.hash_prefix_chunks(packed, toks)
    aligned = hasher.aligned_offsets(lens)
    dev = torch.device("cuda")
    d_off = torch.from_numpy(aligned).to(dev)
    tok = torch.empty(int(aligned[-1]), dtype=torch.int32, device=dev)
    hasher.gen_tokens_device(5, d_off, torch.from_numpy(doc).to(dev), torch.from_numpy(shared).to(dev), tok)
    coff = torch.from_numpy(hasher.chunk_offsets_of_lengths(lens)).to(dev)
    out = torch.empty(int(coff[-1]), dtype=torch.int64, device=dev)
    hasher.hash_prefix_chunks_device(d_off, tok, coff, out)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), want)
    dig = torch.empty_like(out)
    hasher.chunk_digests_device(d_off, tok, coff, dig)
    torch.cuda.synchronize()
    assert not np.array_equal(dig.cpu().numpy(), out.cpu().numpy())  # unchained


@pytest.mark.parametrize("cps,pf,fused", [(3, 0, 0), (3, 0, 1), (3, 1, 0), (3, 1, 1), (2, 4, 1), (4, 0, 1), (1, 2, 1)])
def test_hash_tuning_variants_vs_oracle(oracle, cps, pf, fused):
    """Every K3 tuning (grid, L2 prefetch distance, chain fused into phase 1 with the boundary
    straddlers chained after) gives the oracle's hashes: a random queue, one request spanning
    every CTA range, fewer chunks than CTAs, and empty requests at range boundaries."""
    lib = _capi.lib
    rng = np.random.default_rng(31 + cps + pf)
    cases = [rng.integers(0, 4000, 2000),
             np.array([300, 2_000_000, 0, 0, 700], np.int64),
             np.array([256, 0, 512, 1, 256 * 3], np.int64),
             np.concatenate([np.zeros(50, np.int64), rng.integers(0, 600, 3000), np.zeros(50, np.int64)]),
             # long requests (>= 256 chunks) among short ones, several in one 32-request window
             np.where(rng.random(400) < 0.2, rng.integers(256 * 256, 256 * 1200, 400), rng.integers(0, 9000, 400))]
    try:
        t.check(lib.tsb_hash_set_grid(cps))
        t.check(lib.tsb_hash_set_tuning(pf, fused))
        for lens in cases:
            lens = lens.astype(np.int64)
            offs = np.zeros(len(lens) + 1, np.int64)
            np.cumsum(lens, out=offs[1:])
            toks = oracle.gen_tokens(9, offs, rng.integers(0, 5, len(lens)), lens // 3)
            assert np.array_equal(hasher.hash_prefix_chunks(offs, toks), oracle.hash_prefix_chunks(offs, toks))
    finally:
        t.check(lib.tsb_hash_set_grid(0))
        t.check(lib.tsb_hash_set_tuning(1, 0))  # shipped defaults
