"""Synthetic workloads of BASELINE.json's configs (shapes from the public model configs).

Each workload is a batch of RequestSpecs plus the L2 pool layout that holds their cached
chunks.  Pools model LooGLE-style sharing (many questions over one long document): requests
point at the chunk slots of their document, so the pinned pool stays bounded while every
request still moves its full chunk plan over the host link.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .ingest import LLAMA3_70B, LLAMA31_8B, QWEN25_32B, KVShape
from .tiersim import ClusterConfig, QueueArrays, kv_bytes_per_token


@dataclass
class IngestWorkload:
    name: str
    description: str
    shape: KVShape  # full-head shape (rank shards derived with shape.with_rank)
    queue: QueueArrays
    slots: list  # per request: pool slot of each planned chunk
    pool_slots: int
    config: ClusterConfig = field(default_factory=ClusterConfig)

    def for_rank(self, world: int, rank: int) -> KVShape:
        """KV-head sharding across `world` GPUs, TP-style."""
        if self.shape.kv_heads % world:
            raise ValueError(f"{world} GPUs do not divide {self.shape.kv_heads} KV heads")
        return self.shape.with_rank(world, rank)

    @property
    def chunks(self) -> int:
        return sum(len(s) for s in self.slots)

    def bytes_total(self) -> int:
        """Payload bytes of one pass over the batch, all ranks together."""
        return self.chunks * self.shape.chunk_bytes


def _cluster(shape: KVShape) -> ClusterConfig:
    return ClusterConfig(bytes_per_token=kv_bytes_per_token(shape.layers, shape.kv_heads, shape.head_dim,
                                                            shape.dtype_bytes),
                         block_size_tokens=shape.chunk_tokens)


def _plan_chunks(ctx: int, hit: float, block: int) -> int:
    return int(np.floor(ctx * hit / block))  # cached_token_count floor rule, types.cpp:73-79


def shared_prefix_batch(name, desc, shape, n_req, ctx, hit, query, n_docs) -> IngestWorkload:
    nb = _plan_chunks(ctx, hit, shape.chunk_tokens)
    q = QueueArrays(n_req, id=np.arange(1, n_req + 1), arrival=np.arange(n_req) * 1e-3,
                    context_tokens=np.full(n_req, ctx), query_tokens=np.full(n_req, query),
                    cache_hit_ratio=np.full(n_req, hit), flags=np.zeros(n_req, np.uint8))
    slots = [list(range((r % n_docs) * nb, (r % n_docs) * nb + nb)) for r in range(n_req)]
    return IngestWorkload(name, desc, shape, q, slots, n_docs * nb, _cluster(shape))


def qwen_16x128k() -> IngestWorkload:
    """configs[1]: Qwen2.5-32B KV, 16 x 128K-token prefixes at 90% hit (460 chunks = 30.87 GB each)."""
    return shared_prefix_batch(
        "qwen2.5-32b_16x128k_hit0.9",
        "configs[1]: Qwen2.5-32B KV (64 layers, 8 KV heads, d128, bf16), 16 requests x 128K-token "
        "prefixes at 0.9 hit -> 460 chunks (30.87 GB) each, 493.9 GB per pass; LooGLE-like: the 16 "
        "questions share 2 documents held in a 61.7 GB pinned L2 pool",
        QWEN25_32B, 16, 131072, 0.9, 28, 2)


def llama8b_32k() -> IngestWorkload:
    """configs[0]: Llama-3.1-8B KV, one 32K prefix (128 chunks, 4.29 GB)."""
    return shared_prefix_batch("llama3.1-8b_1x32k", "configs[0]: Llama-3.1-8B KV, one 32K-token prefix, "
                               "128 chunks of 32 MiB", LLAMA31_8B, 1, 32768, 1.0, 28, 1)


def llama70b_32k() -> IngestWorkload:
    """configs[2]: Llama-3-70B KV, one 32K prefix (10.74 GB), KV heads sharded across GPUs."""
    return shared_prefix_batch("llama3-70b_1x32k", "configs[2]: Llama-3-70B KV, one 32K-token prefix "
                               "(10.74 GB), KV heads sharded across the GPUs", LLAMA3_70B, 1, 32768, 1.0, 28, 1)


WORKLOADS = {"qwen16x128k": qwen_16x128k, "llama8b32k": llama8b_32k, "llama70b32k": llama70b_32k}
