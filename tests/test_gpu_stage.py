"""GPU: the real-time load stage (tsb_stage_run) under L1 pressure.

Data parity: every request's pages are checked against the synthetic source pattern before they
are released (verify_seed), and a no-deferral run is compared byte-for-byte with scatter_ref.
Control parity: the TraceEvent-schema log must satisfy the reference's run invariants
(proj/tests/trace_checks.hpp:93-143 -- grant-before-hop, exactly one hop per block, byte
conservation, L1 ledger bound) and the admission order must equal the oracle's pick order.
"""
import numpy as np
import pytest
import torch

import pyoracle as po
from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

from paper_2603_21257_b200 import ingest  # noqa: E402
from paper_2603_21257_b200 import tiersim as t  # noqa: E402
from paper_2603_21257_b200.stage import LoadStage  # noqa: E402

SHAPE = ingest.KVShape(layers=4, kv_heads=8, head_dim=128)
KIND = {"transfer_done": 1, "grant": 2, "compute_done": 3, "dispatch": 4}


def make_queue(n, seed):
    rng = np.random.default_rng(seed)
    ctx = rng.integers(256, 256 * 9, n)
    q = t.QueueArrays(n, id=np.arange(100, 100 + n), arrival=np.round(rng.random(n), 2), context_tokens=ctx,
                      query_tokens=rng.integers(1, 50, n), cache_hit_ratio=rng.choice([0.5, 0.9, 1.0], n),
                      flags=np.ones(n, np.uint8), deadline=5.0 + rng.random(n))
    return q


def slot_lists(q, cfg, n_slots, seed):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(q.n):
        spec = t.RequestSpec(id=int(q.id[i]), context_tokens=int(q.context_tokens[i]),
                             query_tokens=int(q.query_tokens[i]), cache_hit_ratio=float(q.cache_hit_ratio[i]))
        nb = len(t.derive_block_plan(spec, cfg))
        start = int(rng.integers(n_slots))
        out.append([(start + k) % n_slots for k in range(nb)])  # a document's chunks, stored in order
    return out


def check_trace_invariants(tr, chunk_bytes, capacity, plans):
    tr = tr[np.argsort(tr["seq"])]
    grants, dispatch, done = {}, {}, {}
    held, reserved, peak = {}, 0, 0
    for r in tr:
        key = (int(r["request_id"]), int(r["block_index"]))
        if r["kind"] in (KIND["dispatch"], KIND["transfer_done"]) and r["stage"] != 1:
            continue  # online mode also logs compute-stage dispatches (block -1)
        if r["kind"] == KIND["grant"]:
            assert key not in grants, "one grant per block"
            grants[key] = r["seq"]
            reserved += int(r["bytes"])
            held[key[0]] = held.get(key[0], 0) + int(r["bytes"])
            peak = max(peak, reserved)
            assert reserved <= capacity, "L1 ledger bound"
        elif r["kind"] == KIND["dispatch"]:
            assert key in grants and grants[key] < r["seq"], "grant-before-hop"
            assert key not in dispatch, "exactly one hop per block"
            dispatch[key] = r["seq"]
        elif r["kind"] == KIND["transfer_done"]:
            assert key in dispatch and key not in done
            done[key] = r["time"]
            assert r["bytes"] == chunk_bytes
        elif r["kind"] == KIND["compute_done"]:
            reserved -= held.pop(key[0], 0)
    want = {(rid, b) for rid, nb in plans.items() for b in range(nb)}
    assert set(grants) == set(dispatch) == set(done) == want, "byte conservation: every planned block moved once"
    return peak


@pytest.mark.parametrize("mode", ["ce", "bulk", "zerocopy"])
@pytest.mark.parametrize("policy", [t.PolicyKind.Fifo, t.PolicyKind.Lstf])
def test_stage_under_l1_pressure(oracle, mode, policy):
    n_slots, num_pages = 24, 10 * 16  # L1 holds 10 chunks; the batch needs ~50
    pool = ingest.ChunkPool(SHAPE, n_slots)
    pool.fill_synthetic(77)
    l1 = ingest.PagedKVCache(SHAPE, num_pages, max_rows=16, max_chunks=16)
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(4, 8, 128, 2), block_size_tokens=256)
    q = make_queue(12, 3)
    slots = slot_lists(q, cfg, n_slots, 4)
    stage = LoadStage(l1, pool)
    res = stage.run(q, slots, cfg, policy=policy, mode=ingest.MODES[mode], layer_events=True,
                    record_trace=True, verify_seed=77)
    assert res.stats["verify_mismatches"] == 0
    assert res.stats["deferred_chunks"] > 0
    assert res.stats["bytes"] == sum(len(s) for s in slots) * SHAPE.local_chunk_bytes
    assert l1.reserved() == 0 and l1.free_pages() == num_pages
    plans = {int(q.id[i]): len(slots[i]) for i in range(q.n)}
    check_trace_invariants(res.trace, SHAPE.local_chunk_bytes, l1.capacity(), plans)
    # admission order == the oracle's pick order for this policy
    m = t.cost_models_from_config(cfg)
    st, err, tl, tc, pr = oracle.score_queue(q, int(policy), [m.load.slope, m.load.intercept, m.comp.slope,
                                                              m.comp.intercept], cfg)
    order = oracle.sort_order(pr, q.arrival, q.id)
    assert np.array_equal(np.argsort(res.requests["pick_position"]), order)
    # requests become resident in pick order (FIFO grants, single dispatcher)
    loaded = [i for i in order if res.requests["chunks"][i] > 0]  # empty plans are resident at admit
    resident = res.requests["resident_ms"][loaded]
    assert np.all(np.diff(resident) >= 0)
    assert np.all(res.requests["first_layer_ms"] <= res.requests["resident_ms"])


def test_stage_no_pressure_and_errors():
    pool = ingest.ChunkPool(SHAPE, 16)
    pool.fill_synthetic(5)
    l1 = ingest.PagedKVCache(SHAPE, 512, max_rows=8, max_chunks=16)
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(4, 8, 128, 2))
    q = make_queue(4, 9)
    slots = slot_lists(q, cfg, 16, 10)
    stage = LoadStage(l1, pool)
    res = stage.run(q, slots, cfg, mode=ingest.CE, verify_seed=5)
    assert res.stats["verify_mismatches"] == 0 and res.stats["deferred_chunks"] == 0
    assert res.stats["kernel_launches"] > 0
    with pytest.raises(t.ValidationError, match="pool slots for a plan"):
        stage.run(q, [s[:-1] if s else s for s in slots], cfg)
    small = ingest.PagedKVCache(SHAPE, 16, max_rows=8, max_chunks=16)
    with pytest.raises(t.CapacityError, match="can never fit"):
        LoadStage(small, pool).run(q, slots, cfg)
    with pytest.raises(t.MissingDeadline):
        q2 = make_queue(4, 9)
        q2.flags[:] = 0
        stage.run(q2, slots, cfg, policy=t.PolicyKind.Edf)


def test_stage_online_replay_decoupled_semantics():
    """tsb_stage_run_online: arrivals replayed in real time; admission only when the ingest stage
    is idle with no backlog; the best-key pending request wins (engine.cpp:318-339)."""
    pool = ingest.ChunkPool(SHAPE, 24)
    pool.fill_synthetic(3)
    l1 = ingest.PagedKVCache(SHAPE, 64 * 16, max_rows=16, max_chunks=16)
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(4, 8, 128, 2), compute_base=1e-3,
                          compute_per_token=1e-6)
    # request 1 arrives first and occupies the stage; 2..4 arrive together while it runs, so the
    # policy decides among them: SJF-cost must pick the cheapest (fewest chunks) first.
    ctx = np.array([256 * 12, 256 * 9, 256 * 3, 256 * 6])
    q = t.QueueArrays(4, id=np.arange(1, 5), arrival=np.array([0.0, 0.002, 0.002, 0.002]), context_tokens=ctx,
                      query_tokens=np.full(4, 10), cache_hit_ratio=np.ones(4), flags=np.zeros(4, np.uint8))
    slots = [list(range(c // 256)) for c in ctx]
    stage = LoadStage(l1, pool)
    res = stage.run_online(q, slots, cfg, policy=t.PolicyKind.SjfCost)
    r = res.requests
    assert list(np.argsort(r["pick_position"])) == [0, 2, 3, 1]
    assert np.all(r["admit_ms"] >= r["arrival_ms"] - 0.05)
    assert np.all(r["done_ms"] >= r["resident_ms"]) and np.all(r["resident_ms"] > 0)
    assert l1.reserved() == 0
    fifo = stage.run_online(q, slots, cfg, policy=t.PolicyKind.Fifo).requests
    assert list(np.argsort(fifo["pick_position"])) == [0, 1, 2, 3]


def test_stage_synthetic_prefill_overlap():
    """With K6 prefill on a lower-priority stream, ingest of later requests overlaps earlier
    prefills: the batch finishes well before sum(ingest) + sum(prefill)."""
    shape = ingest.KVShape(layers=8, kv_heads=8, head_dim=128)
    pool = ingest.ChunkPool(shape, 64)
    pool.fill_synthetic(1)
    l1 = ingest.PagedKVCache(shape, 64 * 16, max_rows=8, max_chunks=64)
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(8, 8, 128, 2), compute_base=2e-3,
                          compute_per_token=2e-6)
    q = t.QueueArrays(6, id=np.arange(6), arrival=np.zeros(6), context_tokens=np.full(6, 256 * 40),
                      query_tokens=np.full(6, 500), cache_hit_ratio=np.ones(6), flags=np.zeros(6, np.uint8))
    slots = [list(range(40))] * 6
    stage = LoadStage(l1, pool)
    res = stage.run(q, slots, cfg, mode=ingest.CE, layer_events=True, prefill=True, verify_seed=1)
    assert res.stats["verify_mismatches"] == 0
    r = res.requests
    assert np.all(r["done_ms"] >= r["resident_ms"])
    prefill_s = cfg.compute_base + cfg.compute_per_token * 500
    assert r["done_ms"].max() * 1e-3 >= 6 * prefill_s * 0.9
    # the stage's 128 MiB CE group cap under a prefill is scoped to the run; a caller's cap stays
    assert l1.ce_group_bytes == 0
    l1.ce_group_bytes = 3 << 20
    res = stage.run(q, slots, cfg, mode=ingest.CE, layer_events=True, prefill=True, verify_seed=1)
    assert res.stats["verify_mismatches"] == 0 and l1.ce_group_bytes == 3 << 20


@pytest.mark.parametrize("layer_events", [False, True])
def test_stage_reuse_l1_replicates_resident_chunks(layer_events):
    """reuse_l1: requests reading the same document chunks get them from a live holder's pages
    (K8, HBM -> HBM) instead of the host link; every page is still verified, the holders' pages are
    released only after the copies, and the result equals the link-only run."""
    shape = ingest.KVShape(layers=4, kv_heads=8, head_dim=128)
    pool = ingest.ChunkPool(shape, 24)
    pool.fill_synthetic(9)
    l1 = ingest.PagedKVCache(shape, 20 * 16, max_rows=16, max_chunks=16)  # L1 pressure: deferral
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(4, 8, 128, 2), compute_base=1e-4,
                          compute_per_token=1e-7)
    n = 8
    q = t.QueueArrays(n, id=np.arange(1, n + 1), arrival=np.arange(n) * 1e-3, context_tokens=np.full(n, 256 * 6),
                      query_tokens=np.full(n, 10), cache_hit_ratio=np.ones(n), flags=np.zeros(n, np.uint8))
    docs = [list(range(0, 6)), list(range(10, 16)), list(range(3, 9))]  # doc 2 overlaps doc 0
    slots = [docs[i % 3] for i in range(n)]
    stage = LoadStage(l1, pool)
    base = stage.run(q, slots, cfg, prefill=True, layer_events=layer_events, verify_seed=9)
    res = stage.run(q, slots, cfg, prefill=True, layer_events=layer_events, verify_seed=9, reuse_l1=True)
    assert base.stats["verify_mismatches"] == 0 and res.stats["verify_mismatches"] == 0
    assert base.stats["reused_chunks"] == 0 and res.stats["reused_chunks"] >= 12
    assert res.stats["bytes"] == base.stats["bytes"] == n * 6 * shape.local_chunk_bytes
    assert l1.reserved() == 0 and l1.free_pages() == l1.num_pages
    r = res.requests
    assert np.all(r["done_ms"] >= r["resident_ms"]) and np.all(r["resident_ms"] >= r["first_layer_ms"])


@pytest.mark.parametrize("control", [t.ControlMode.Decoupled, t.ControlMode.Coupled])
def test_stage_online_reuse_l1(control):
    """Online replay with reuse_l1: requests arriving over time that share document chunks get
    them from a live holder's pages (K8) instead of the host link, under L1 pressure (deferral);
    every page is verified, the trace keeps the reference invariants (grant-before-hop, one hop
    per block, byte conservation, ledger bound), holders' pages are released only after the
    copies that read them, and the allocator ends empty."""
    pool = ingest.ChunkPool(SHAPE, 24)
    pool.fill_synthetic(21)
    l1 = ingest.PagedKVCache(SHAPE, 16 * 16, max_rows=16, max_chunks=16)  # 16 chunks of pages
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(4, 8, 128, 2), compute_base=2e-3,
                          compute_per_token=1e-7, control_mode=control)
    n = 10
    q = t.QueueArrays(n, id=np.arange(1, n + 1), arrival=np.arange(n) * 4e-4, context_tokens=np.full(n, 256 * 6),
                      query_tokens=np.full(n, 10), cache_hit_ratio=np.ones(n), flags=np.zeros(n, np.uint8))
    docs = [list(range(0, 6)), list(range(10, 16)), list(range(3, 9))]  # doc 2 overlaps doc 0
    slots = [docs[i % 3] for i in range(n)]
    stage = LoadStage(l1, pool)
    base = stage.run_online(q, slots, cfg, verify_seed=21, record_trace=True)
    res = stage.run_online(q, slots, cfg, verify_seed=21, record_trace=True, reuse_l1=True)
    for r in (base, res):
        assert r.stats["verify_mismatches"] == 0
        assert r.stats["bytes"] == n * 6 * SHAPE.local_chunk_bytes
        check_trace_invariants(r.trace, SHAPE.local_chunk_bytes, l1.capacity(), {i + 1: 6 for i in range(n)})
    assert base.stats["reused_chunks"] == 0
    if control == t.ControlMode.Decoupled:
        assert res.stats["reused_chunks"] > 0
    assert l1.reserved() == 0 and l1.free_pages() == l1.num_pages
    r = res.requests
    assert np.all(r["done_ms"] >= r["resident_ms"]) and np.all(r["resident_ms"] >= r["first_layer_ms"])


def test_copy_chunks_api(oracle):
    """tsb_l1_copy_chunks (K8) against scatter_ref: chunks ingested into row A, replicated into row B."""
    import ctypes as C

    from paper_2603_21257_b200 import _capi

    shape = ingest.KVShape(layers=3, kv_heads=8, head_dim=128)
    pool = ingest.ChunkPool(shape, 6)
    pool.fill_synthetic(4)
    l1 = ingest.PagedKVCache(shape, 12 * 16, max_rows=3, max_chunks=6)
    l1.arena.zero_()
    cb = shape.page_bytes * 16
    ra = [l1.request(1, c, cb)[1] for c in range(4)][0]
    rb = [l1.request(2, c, cb)[1] for c in range(4)][0]
    l1.sync_block_table()
    ingest.ingest(l1, pool, ingest.items_numpy([5, 1, 2, 0], [ra] * 4, range(4)))
    items = (_capi.PageCopy * 4)(*[_capi.PageCopy(ra, c, rb, 3 - c) for c in range(4)])
    t.check(_capi.lib.tsb_l1_copy_chunks(l1.handle, items, 4, 0, 3, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = oracle.scatter_ref(shape, pool.slot_view(0, 6),
                              ingest.items_numpy([5, 1, 2, 0, 0, 2, 1, 5], [ra] * 4 + [rb] * 4, [0, 1, 2, 3] * 2),
                              l1.block_table(), l1.num_pages)
    assert np.array_equal(l1.arena.cpu().numpy(), want)
    bad = (_capi.PageCopy * 1)(_capi.PageCopy(ra, 0, 7, 0))
    with pytest.raises(t.ValidationError, match="outside the block table"):
        t.check(_capi.lib.tsb_l1_copy_chunks(l1.handle, bad, 1, 0, 3, None))
