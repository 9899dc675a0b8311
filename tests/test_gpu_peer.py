"""GPU: the peer-HBM tier -- chunk pools resident in GPU memory.

A device pool has the L2 slot layout ([L][2][C][H][D] per slot) but lives in HBM: this GPU's,
or a peer's reached over NVLink through peer access / CUDA IPC.  The ingest kernels read it with
the same addressing as a host pool, so parity is the same scatter_ref oracle.  The box has one
GPU: the peer case is exercised as two processes sharing cuda:0 through an exported IPC handle
(the code path a second GPU takes, minus the NVLink hop).
"""
import os
import socket

import numpy as np
import pytest
import torch

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

from paper_2603_21257_b200 import ingest  # noqa: E402
from paper_2603_21257_b200 import tiersim as t  # noqa: E402
from test_gpu_parity import SMALL, build_scenario  # noqa: E402


def host_twin(shape, n_slots, seed):
    """Host pool with the same synthetic bytes (the pattern is a function of seed and word index)."""
    p = ingest.ChunkPool(shape, n_slots)
    p.fill_synthetic(seed)
    return p


@pytest.mark.parametrize("tp", [(1, 0), (2, 1), (8, 5)])
@pytest.mark.parametrize("mode", ["auto", "zerocopy", "bulk"])
def test_device_pool_ingest_bit_exact(oracle, tp, mode):
    shape = SMALL.with_rank(*tp)
    dpool = ingest.ChunkPool.create_device(shape, 8)
    dpool.fill_synthetic(17)
    assert dpool.on_device and dpool.device == 0
    pool, l1, items = build_scenario(shape, pool=dpool)
    ingest.ingest(l1, pool, items, mode=ingest.MODES[mode])
    torch.cuda.synchronize()
    twin = host_twin(shape, 8, 17)  # keep alive: slot_view aliases its pinned memory
    want = oracle.scatter_ref(shape, twin.slot_view(0, 8), items, l1.block_table(), l1.num_pages)
    assert np.array_equal(l1.arena.cpu().numpy(), want)
    assert ingest.verify_synthetic(l1, pool, items, seed=17) == 0


def test_wrapped_tensor_pool_per_layer_events(oracle):
    """A torch CUDA tensor of random bytes as the pool; per-layer ingest with events."""
    g = torch.Generator(device="cuda").manual_seed(3)
    buf = torch.randint(0, 256, (6 * SMALL.chunk_bytes,), dtype=torch.uint8, device="cuda", generator=g)
    pool = ingest.ChunkPool.wrap_device(SMALL, buf)
    assert pool.n_slots == 6
    _, l1, items = build_scenario(SMALL, pool=pool)
    s = torch.cuda.Stream()
    evs = [torch.cuda.Event() for _ in range(SMALL.layers)]
    with torch.cuda.stream(s):
        ingest.ingest(l1, pool, items, mode=ingest.ZEROCOPY, stream=s, layer_events=evs)
    evs[-1].synchronize()
    want = oracle.scatter_ref(SMALL, buf.cpu().numpy(), items, l1.block_table(), l1.num_pages)
    assert np.array_equal(l1.arena.cpu().numpy(), want)


def test_device_pool_errors_fail_loudly():
    pool = ingest.ChunkPool.create_device(SMALL, 2)
    _, l1, items = build_scenario(SMALL, pool=pool)
    with pytest.raises(t.Unsupported, match="CE mode reads host pools"):
        ingest.ingest(l1, pool, items, mode=ingest.CE)
    with pytest.raises(TypeError):
        pool.slot_view(0)
    with pytest.raises(t.ValidationError, match="n_slots"):
        ingest.ChunkPool.wrap_device(SMALL, torch.empty(SMALL.chunk_bytes, dtype=torch.uint8, device="cuda"),
                                     n_slots=0)
    hp = ingest.ChunkPool(SMALL, 1)
    with pytest.raises(t.ValidationError, match="only tsb_pool_create_device"):
        hp.ipc_handle()
    ingest.enable_peer_access(0, 0)  # same device: a no-op


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        torch.cuda.set_device(0)
        if rank == 0:  # the owner: an HBM chunk pool other processes read
            pool = ingest.ChunkPool.create_device(SMALL, 8)
            pool.fill_synthetic(29)
            msg = [pool.ipc_handle()]
            dist.broadcast_object_list(msg, src=0)
            dist.barrier()  # the reader is done before the owner frees the memory
            pool.close()
            q.put((rank, "ok"))
        else:
            msg = [None]
            dist.broadcast_object_list(msg, src=0)
            pool = ingest.ChunkPool.open_ipc(SMALL, msg[0], n_slots=8, owner_device=0)
            _, l1, items = build_scenario(SMALL, pool=pool)
            for mode in (ingest.ZEROCOPY, ingest.BULK):
                l1.arena.zero_()
                ingest.ingest(l1, pool, items, mode=mode)
                torch.cuda.synchronize()
                bad = ingest.verify_synthetic(l1, pool, items, seed=29)
                if bad:
                    q.put((rank, f"mode {mode}: {bad} mismatching words"))
                    break
            else:
                q.put((rank, "ok"))
            pool.close()
            dist.barrier()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_ipc_pool_across_processes():
    """Rank 0 owns an HBM pool and exports it; rank 1 maps it (cudaIpcOpenMemHandle) and ingests
    from it into its own paged L1.  Handles travel over gloo: plumbing, not a data path."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert results == {0: "ok", 1: "ok"}, results


def test_tiered_ingest_mixes_hbm_tier_and_host_pool(oracle):
    """tsb_ingest_tiered: negative slots come from the HBM tier, the rest over the host link; both
    pools hold the same synthetic pattern per slot index, so the pages equal scatter_ref over the
    host pool at |slot|.  Every mode of the host part, full heads and a TP shard."""
    from test_gpu_parity import SMALL

    for tp in ((1, 0), (4, 1)):
        shape = SMALL.with_rank(*tp)
        host = ingest.ChunkPool(SMALL, 8)
        host.fill_synthetic(21)
        tier = ingest.ChunkPool.create_device(SMALL, 8)
        tier.fill_synthetic(21)
        for mode in ("auto", "ce", "zerocopy", "bulk"):
            num_pages = 160
            arena = torch.zeros(shape.layers * 2 * num_pages * 16 * shape.heads_local * 128 * 2, dtype=torch.uint8,
                                device="cuda")
            l1 = ingest.PagedKVCache(shape, num_pages, max_rows=2, max_chunks=10, arena=arena)
            rows = [l1.request(3, c, shape.page_bytes * 16)[1] for c in range(9)]
            l1.sync_block_table()
            content = [5, 0, 7, 7, 1, 2, 3, 6, 4]
            slots = [s if c % 3 else ~s for c, s in enumerate(content)]  # every third chunk from the tier
            items = ingest.items_numpy(slots, rows, range(9))
            evs = [torch.cuda.Event() for _ in range(shape.layers)]
            ingest.ingest_tiered(l1, host, tier, items, mode=ingest.MODES[mode], layer_events=evs)
            evs[-1].synchronize()
            want = oracle.scatter_ref(shape, host.slot_view(0, 8), ingest.items_numpy(content, rows, range(9)),
                                      l1.block_table(), num_pages)
            assert np.array_equal(arena.cpu().numpy(), want), (tp, mode)
            l1.close()
    with pytest.raises(t.ValidationError, match="HBM tier"):
        ingest.ingest_tiered(l1, host, None, items)


def test_stage_with_hbm_tier_verifies_every_page():
    from paper_2603_21257_b200.stage import LoadStage

    shape = ingest.KVShape(layers=4, kv_heads=8, head_dim=128)
    host = ingest.ChunkPool(shape, 12)
    host.fill_synthetic(8)
    tier = ingest.ChunkPool.create_device(shape, 6)
    tier.fill_synthetic(8)
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(4, 8, 128, 2), block_size_tokens=256)
    q = t.QueueArrays(3, id=np.array([1, 2, 3]), arrival=np.array([0.0, 0.1, 0.2]),
                      context_tokens=np.array([256 * 5, 256 * 6, 256 * 4]), query_tokens=np.full(3, 10),
                      cache_hit_ratio=np.ones(3), flags=np.zeros(3, np.uint8))
    slots = [[~0, ~1, 2, 3, 4], [5, ~2, 6, ~3, 7, 8], [~4, ~5, 9, 10]]  # negative: chunk resident in the HBM tier
    l1 = ingest.PagedKVCache(shape, 10 * 16, max_rows=4, max_chunks=8)  # 10 chunks of pages: deferral
    stage = LoadStage(l1, host)
    with pytest.raises(t.ValidationError):
        stage.run(q, slots, cfg, verify_seed=8)  # no tier set: negative slots are out of range
    stage.set_hbm_tier(tier)
    res = stage.run(q, slots, cfg, verify_seed=8)
    assert res.stats["verify_mismatches"] == 0
    assert res.stats["bytes"] == 15 * shape.local_chunk_bytes
    assert res.stats["deferred_chunks"] > 0


def test_tiered_ingest_all_tier_and_empty(oracle):
    """All chunks from the HBM tier (no L2 pool given) and an empty call: fences still fire."""
    from test_gpu_parity import SMALL

    host = ingest.ChunkPool(SMALL, 4)
    host.fill_synthetic(5)
    tier = ingest.ChunkPool.create_device(SMALL, 4)
    tier.fill_synthetic(5)
    arena = torch.zeros(SMALL.layers * 2 * 64 * 16 * 8 * 128 * 2, dtype=torch.uint8, device="cuda")
    l1 = ingest.PagedKVCache(SMALL, 64, max_rows=1, max_chunks=4, arena=arena)
    rows = [l1.request(1, c, SMALL.page_bytes * 16)[1] for c in range(3)]
    l1.sync_block_table()
    evs = [torch.cuda.Event() for _ in range(SMALL.layers)]
    ingest.ingest_tiered(l1, None, tier, ingest.items_numpy([~3, ~1, ~2], rows, [0, 1, 2]), layer_events=evs)
    for e in evs:
        e.synchronize()
    want = oracle.scatter_ref(SMALL, host.slot_view(0, 4), ingest.items_numpy([3, 1, 2], rows, [0, 1, 2]),
                              l1.block_table(), 64)
    assert np.array_equal(arena.cpu().numpy(), want)
    evs2 = [torch.cuda.Event() for _ in range(SMALL.layers)]
    ingest.ingest_tiered(l1, None, None, ingest.items_numpy([], [], []), layer_events=evs2)
    for e in evs2:
        e.synchronize()
    with pytest.raises(t.ValidationError, match="no L2 pool"):
        ingest.ingest_tiered(l1, None, tier, ingest.items_numpy([0], [rows[0]], [0]))
