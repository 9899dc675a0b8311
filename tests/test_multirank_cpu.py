"""World-size-2 gloo tests of the N>1 path on CPU: KV-head sharding, the shared pool segment,
and max-over-ranks timing.  The device ingest itself is covered by the sharded GPU parity tests."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import pyoracle as po
        from paper_2603_21257_b200.ingest import KVShape
        from paper_2603_21257_b200.multirank import SharedSegment, head_shards, reduce_timing

        full = KVShape(layers=3, kv_heads=8, head_dim=16, chunk_tokens=64, page_tokens=16)
        shard = head_shards(full.kv_heads, world)[rank]
        shape = full.with_rank(world, rank)
        assert (shard.head_lo, shard.head_hi) == (rank * 8 // world, (rank + 1) * 8 // world)

        # one pool segment for the "box": rank 0 creates and fills it, every rank maps it
        n_slots = 4
        nbytes = n_slots * full.chunk_bytes
        seg = SharedSegment(f"tsb_test_{port}", nbytes, rank, dist.barrier)
        view = np.frombuffer(seg.mm, dtype=np.uint8)
        if rank == 0:
            view[:] = po.synth_fill(3, 0, nbytes // 8).view(np.uint8)
        dist.barrier()
        seg.unlink()  # every rank has mapped it: the name goes, the mappings stay
        dist.barrier()
        assert not os.path.exists(seg.path)
        assert np.array_equal(view[:64], po.synth_fill(3, 0, 8).view(np.uint8))

        # each rank scatters its head slice; identical block tables on every rank
        items = np.array([(2, 0, 0), (0, 0, 1), (3, 0, 2)],
                         dtype=[("src_slot", np.int64), ("bt_row", np.int32), ("chunk_index", np.int32)])
        bt = np.arange(12, dtype=np.int32)[::-1].copy().reshape(1, 12)
        local = po.scatter_ref(shape, view, items, bt, 12).reshape(3, 2, 12, 16, 8 // world, 32)
        gathered = [torch.zeros(local.shape, dtype=torch.uint8) for _ in range(world)] if rank == 0 else None
        dist.gather(torch.from_numpy(local.view(np.uint8).copy()), gathered, dst=0)

        dev_s, wall_s, total = reduce_timing(dist, 1.0 + rank, 2.0 + rank, 100.0 * (rank + 1))
        if rank == 0:
            # the union of the rank slices is the unsharded scatter, heads concatenated
            full_arena = po.scatter_ref(full, view, items, bt, 12).reshape(3, 2, 12, 16, 8, 32)
            # bytes per head row: head_dim * dtype_bytes = 32 -> local layout [..., heads_local, 32 B]
            cat = np.concatenate([g.numpy() for g in gathered], axis=4)
            q.put((bool(np.array_equal(cat, full_arena)), dev_s, wall_s, total))
        dist.barrier()
        seg.close(unlink=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_head_sharded_ingest_union_equals_full_and_max_timing(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok, dev_s, wall_s, total = q.get(timeout=90)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok
    assert (dev_s, wall_s) == (float(world), float(world + 1))  # max over ranks
    assert total == sum(100.0 * (r + 1) for r in range(world))  # bytes summed over ranks


def test_head_shards_validation():
    sys.path.insert(0, str(ROOT))
    from paper_2603_21257_b200.multirank import head_shards

    assert [s.head_hi - s.head_lo for s in head_shards(8, 8)] == [1] * 8
    with pytest.raises(ValueError):
        head_shards(8, 3)
