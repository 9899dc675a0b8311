"""Prefix chunk hasher (K3) -- tsb_hash_prefix_chunks*.

Chained per-256-token-chunk hashes: hash c of request r names the whole token prefix
[0, 256(c+1)), so an L2 lookup can find how many leading chunks are already stored.  Definition
frozen in oracle/tsb_oracle.c (orc_hash_prefix_chunks), built on the reference's FNV-1a-64
constants (engine.cpp:500-534).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from ._capi import lib
from .tiersim import check


def chunk_offsets(offsets: np.ndarray) -> np.ndarray:
    lens = np.diff(np.asarray(offsets, dtype=np.int64))
    out = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens // 256, out=out[1:])
    return out


def hash_prefix_chunks(offsets: np.ndarray, tokens: np.ndarray, stream=None) -> np.ndarray:
    """Host arrays in, host hashes out (H2D, kernel, D2H inside)."""
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    tokens = np.ascontiguousarray(tokens, dtype=np.int32)
    n_req = len(offsets) - 1
    total = int(chunk_offsets(offsets)[-1])
    out = np.empty(max(total, 1), dtype=np.uint64)
    n = C.c_int64()
    s = (stream or torch.cuda.current_stream()).cuda_stream
    check(lib.tsb_hash_prefix_chunks(s, n_req, offsets.ctypes.data, tokens.ctypes.data, out.ctypes.data, C.byref(n)))
    return out[: n.value]


def hash_prefix_chunks_device(offsets: torch.Tensor, tokens: torch.Tensor, coffsets: torch.Tensor,
                              out: torch.Tensor, stream=None) -> torch.Tensor:
    s = (stream or torch.cuda.current_stream()).cuda_stream
    check(lib.tsb_hash_prefix_chunks_device(s, offsets.numel() - 1, offsets.data_ptr(), tokens.data_ptr(),
                                            coffsets.data_ptr(), out.data_ptr()))
    return out


def chunk_digests_device(offsets: torch.Tensor, tokens: torch.Tensor, coffsets: torch.Tensor, out: torch.Tensor,
                         stream=None) -> torch.Tensor:
    """K3 phase 1 alone: every full chunk's own digest (tsb_hash_chunk_digests_device)."""
    s = (stream or torch.cuda.current_stream()).cuda_stream
    check(lib.tsb_hash_chunk_digests_device(s, coffsets.numel() - 1, offsets.data_ptr(), tokens.data_ptr(),
                                            coffsets.data_ptr(), out.data_ptr()))
    return out


def aligned_offsets(lengths: np.ndarray, align_tokens: int = 4) -> np.ndarray:
    """Request starts padded to `align_tokens` (4 int32 = 16 bytes) with gaps between requests:
    the layout the device hasher reads fastest; chunk counts still come from the true lengths."""
    lengths = np.asarray(lengths, np.int64)
    padded = (lengths + align_tokens - 1) // align_tokens * align_tokens
    offs = np.zeros(len(lengths) + 1, np.int64)
    np.cumsum(padded, out=offs[1:])
    return offs


def chunk_offsets_of_lengths(lengths: np.ndarray) -> np.ndarray:
    lengths = np.asarray(lengths, np.int64)
    co = np.zeros(len(lengths) + 1, np.int64)
    np.cumsum(lengths // 256, out=co[1:])
    return co


class PrefixIndex:
    """L2 chunk index on the GPU (K7): chained chunk hash -> L2 pool slot (tsb_index_*).

    lookup() returns, per request, the matched prefix in chunks and the pool slots of those
    chunks -- the real-prefix replacement for the reference's synthetic cache_hit_ratio."""

    def __init__(self, capacity: int, device: int = 0):
        h = C.c_void_p()
        check(lib.tsb_index_create(device, int(capacity), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) and lib is not None:  # lib is None during interpreter exit
            lib.tsb_index_destroy(self._h)
            self._h = None

    __del__ = close

    @property
    def capacity(self) -> int:
        return lib.tsb_index_capacity(self._h)

    def insert(self, hashes: np.ndarray, slots: np.ndarray, stream=None):
        hashes = np.ascontiguousarray(hashes, np.uint64)
        slots = np.ascontiguousarray(slots, np.int64)
        s = (stream or torch.cuda.current_stream()).cuda_stream
        check(lib.tsb_index_insert(self._h, s, len(hashes), hashes.ctypes.data, slots.ctypes.data))

    def insert_device(self, hashes: torch.Tensor, slots: torch.Tensor, stream=None):
        s = (stream or torch.cuda.current_stream()).cuda_stream
        check(lib.tsb_index_insert_device(self._h, s, hashes.numel(), hashes.data_ptr(), slots.data_ptr()))

    def lookup_device(self, chunk_offs: torch.Tensor, hashes: torch.Tensor, slots_out: torch.Tensor,
                      matched_out: torch.Tensor, stream=None):
        s = (stream or torch.cuda.current_stream()).cuda_stream
        check(lib.tsb_index_lookup_device(self._h, s, chunk_offs.numel() - 1, chunk_offs.data_ptr(),
                                          hashes.data_ptr(), slots_out.data_ptr(), matched_out.data_ptr()))

    def erase_device(self, hashes: torch.Tensor, stream=None):
        s = (stream or torch.cuda.current_stream()).cuda_stream
        check(lib.tsb_index_erase_device(self._h, s, hashes.numel(), hashes.data_ptr()))

    def lookup(self, chunk_offs: np.ndarray, hashes: np.ndarray, stream=None):
        chunk_offs = np.ascontiguousarray(chunk_offs, np.int64)
        hashes = np.ascontiguousarray(hashes, np.uint64)
        n_req = len(chunk_offs) - 1
        slots = np.empty(max(len(hashes), 1), np.int64)
        matched = np.empty(max(n_req, 1), np.int64)
        s = (stream or torch.cuda.current_stream()).cuda_stream
        check(lib.tsb_index_lookup(self._h, s, n_req, chunk_offs.ctypes.data, hashes.ctypes.data,
                                   slots.ctypes.data, matched.ctypes.data))
        return matched[:n_req], slots[: len(hashes)]

    def clear(self, stream=None):
        check(lib.tsb_index_clear(self._h, (stream or torch.cuda.current_stream()).cuda_stream))

    def compact(self, stream=None) -> int:
        """Rebuild without erase tombstones; returns how many were reclaimed."""
        n = C.c_int64()
        check(lib.tsb_index_compact(self._h, (stream or torch.cuda.current_stream()).cuda_stream, C.byref(n)))
        return n.value

    def stats(self, stream=None):
        live, full = C.c_int64(), C.c_int64()
        s = (stream or torch.cuda.current_stream()).cuda_stream
        check(lib.tsb_index_stats(self._h, s, C.byref(live), C.byref(full)))
        return live.value, full.value


def hit_ratio_for_match(context_tokens: int, matched_chunks: int, block: int = 256) -> float:
    """A cache_hit_ratio whose floor rule (types.cpp:73-79) yields exactly matched_chunks."""
    if matched_chunks * block >= context_tokens:
        return 1.0
    return (matched_chunks * block + block / 2) / context_tokens


def gen_tokens_device(seed: int, offsets: torch.Tensor, doc: torch.Tensor, shared_len: torch.Tensor,
                      out: torch.Tensor, stream=None) -> torch.Tensor:
    s = (stream or torch.cuda.current_stream()).cuda_stream
    check(lib.tsb_gen_tokens_device(s, int(seed), offsets.numel() - 1, offsets.data_ptr(), doc.data_ptr(),
                                    shared_len.data_ptr(), out.data_ptr()))
    return out
