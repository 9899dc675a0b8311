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


def gen_tokens_device(seed: int, offsets: torch.Tensor, doc: torch.Tensor, shared_len: torch.Tensor,
                      out: torch.Tensor, stream=None) -> torch.Tensor:
    s = (stream or torch.cuda.current_stream()).cuda_stream
    check(lib.tsb_gen_tokens_device(s, int(seed), offsets.numel() - 1, offsets.data_ptr(), doc.data_ptr(),
                                    shared_len.data_ptr(), out.data_ptr()))
    return out
