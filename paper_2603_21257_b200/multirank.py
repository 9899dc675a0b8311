"""One process per GPU: KV-head sharding, the shared L2 pool segment, and max-over-ranks timing.

The ingest path shards by KV head, TP-style: rank r of N keeps heads
[r*H/N, (r+1)*H/N) of every (layer, K/V, token) and reads only that slice over its own host link
-- from a rank-local pinned pool on its GPU's NUMA node holding just those heads (the default,
bench.py make_pool), or strided out of full chunks in one /dev/shm segment shared by all ranks
(SharedSegment).  Ranks never exchange data: torch.distributed is used for barriers and for the
max-over-ranks reduction of timings only.
"""
from __future__ import annotations

import mmap
import os
from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    head_lo: int
    head_hi: int


def head_shards(kv_heads: int, world: int) -> list:
    if world < 1 or kv_heads % world:
        raise ValueError(f"{world} ranks do not divide {kv_heads} KV heads")
    h = kv_heads // world
    return [Shard(r, world, r * h, (r + 1) * h) for r in range(world)]


def reduce_timing(dist, dev_s: float, wall_s: float, local_bytes: float, device=None):
    """Returns (max device seconds, max wall seconds, total bytes) over ranks (single rank: as is)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return dev_s, wall_s, local_bytes
    t = torch.tensor([dev_s, wall_s], dtype=torch.float64, device=device)
    b = torch.tensor([local_bytes], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(b, op=dist.ReduceOp.SUM)
    return float(t[0]), float(t[1]), float(b[0])


class SharedSegment:
    """A /dev/shm file mapped MAP_SHARED by every rank (rank 0 creates it)."""

    def __init__(self, name: str, nbytes: int, rank: int, barrier):
        self.path = f"/dev/shm/{name}"
        self.nbytes = nbytes
        if rank == 0:
            with open(self.path, "wb") as f:
                f.truncate(nbytes)
        barrier()
        self.fd = os.open(self.path, os.O_RDWR)
        self.mm = mmap.mmap(self.fd, nbytes, mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)
        self.rank = rank

    @staticmethod
    def fits(nbytes: int) -> bool:
        try:
            st = os.statvfs("/dev/shm")
        except OSError:
            return False
        return st.f_bavail * st.f_frsize > nbytes * 1.05

    def address(self) -> int:
        import ctypes

        return ctypes.addressof(ctypes.c_char.from_buffer(self.mm))

    def unlink(self):
        """Rank 0 removes the /dev/shm name once every rank has mapped it: the mappings stay valid
        and the memory is returned when the last process exits, so no segment outlives the run."""
        if self.rank == 0 and os.path.exists(self.path):
            os.unlink(self.path)

    def close(self, unlink: bool = False):
        try:
            self.mm.close()
        except BufferError:
            pass  # a registered view is still alive; the mapping dies with the process
        os.close(self.fd)
        if unlink and self.rank == 0 and os.path.exists(self.path):
            os.unlink(self.path)
