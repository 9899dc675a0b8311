"""L2 pinned chunk pool, L1 paged KV cache + block_table, and the L2->L1 ingest (K1/K1b/CE+K2).

Python face of tsb_pool_* / tsb_l1_* / tsb_ingest*.  The reference models this hop only as a
duration (engine.cpp:206-207, pcie_dispatch engine.cpp:427-446); here it moves real bytes:
LMCache-style chunks [layer][K/V][token][kv_head][dim] in pinned host memory are scattered
into vLLM-style paged HBM blocks [2][num_pages][page_tokens][kv_heads_local][head_dim] per
layer through the block table.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _capi as capi
from ._capi import lib
from .tiersim import Tier, check

ZEROCOPY, BULK, CE, AUTO = capi.INGEST_ZEROCOPY, capi.INGEST_BULK, capi.INGEST_CE, capi.INGEST_AUTO
CE_DIRECT = capi.INGEST_CE_DIRECT
MODES = {"auto": AUTO, "zerocopy": ZEROCOPY, "bulk": BULK, "ce": CE, "ce_direct": CE_DIRECT}
# Page layouts of the L1 arena (tsb_kv_layout): the consumer's KV-cache layout.
LAYOUT_FLASH_ATTN, LAYOUT_FLASHINFER_NHD, LAYOUT_FLASHINFER_HND = 0, 1, 2
LAYOUTS = {"flash_attn": LAYOUT_FLASH_ATTN, "flashinfer_nhd": LAYOUT_FLASHINFER_NHD,
           "flashinfer_hnd": LAYOUT_FLASHINFER_HND}


@dataclass(frozen=True)
class KVShape:
    layers: int
    kv_heads: int
    head_dim: int
    dtype_bytes: int = 2
    chunk_tokens: int = 256
    page_tokens: int = 16
    tp_size: int = 1
    tp_rank: int = 0

    def struct(self) -> capi.KvShape:
        return capi.KvShape(self.layers, self.kv_heads, self.head_dim, self.dtype_bytes, self.chunk_tokens,
                            self.page_tokens, self.tp_size, self.tp_rank)

    def info(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.tsb_kv_shape_info(C.byref(self.struct()), C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    @property
    def chunk_bytes(self) -> int:
        return self.info()[0]

    @property
    def page_bytes(self) -> int:
        """Local bytes of one page across all layers (K and V, this rank's heads)."""
        return self.info()[1]

    @property
    def local_chunk_bytes(self) -> int:
        return self.info()[2]

    @property
    def heads_local(self) -> int:
        return self.kv_heads // self.tp_size

    @property
    def pages_per_chunk(self) -> int:
        return self.chunk_tokens // self.page_tokens

    def with_rank(self, tp_size: int, tp_rank: int) -> "KVShape":
        return KVShape(self.layers, self.kv_heads, self.head_dim, self.dtype_bytes, self.chunk_tokens,
                       self.page_tokens, tp_size, tp_rank)


# Model shapes of BASELINE.json (public configs).
LLAMA31_8B = KVShape(layers=32, kv_heads=8, head_dim=128)
QWEN25_32B = KVShape(layers=64, kv_heads=8, head_dim=128)
LLAMA3_70B = KVShape(layers=80, kv_heads=8, head_dim=128)


def _stream(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def device_numa_node(device: int) -> int:
    """NUMA node of a GPU's PCIe root (-1 if the platform does not say)."""
    return lib.tsb_device_numa_node(int(device))


class ChunkPool:
    """L2 tier: pinned + portable + mapped host memory, one full chunk per slot."""

    def __init__(self, shape: KVShape, n_slots: int):
        self.shape = shape
        h = C.c_void_p()
        check(lib.tsb_pool_create(C.byref(shape.struct()), int(n_slots), C.byref(h)))
        self._h = h
        self.n_slots = n_slots
        self.chunk_bytes = lib.tsb_pool_chunk_bytes(h)

    @classmethod
    def register(cls, shape: KVShape, host_ptr: int, n_slots: int, keepalive=None) -> "ChunkPool":
        """Page-lock caller memory (e.g. a /dev/shm segment every per-GPU process maps) as the pool."""
        self = cls.__new__(cls)
        self.shape = shape
        h = C.c_void_p()
        check(lib.tsb_pool_register(C.byref(shape.struct()), int(host_ptr), int(n_slots), C.byref(h)))
        self._h = h
        self.n_slots = n_slots
        self.chunk_bytes = lib.tsb_pool_chunk_bytes(h)
        self._keepalive = keepalive
        return self

    @classmethod
    def create_numa(cls, shape: KVShape, n_slots: int, numa_node: int) -> "ChunkPool":
        """Pinned pool whose pages live on NUMA node `numa_node` (tsb_pool_create_numa; -1 = the
        default policy).  Use device_numa_node(gpu) to put each GPU's pool on its own socket."""
        h = C.c_void_p()
        check(lib.tsb_pool_create_numa(C.byref(shape.struct()), int(n_slots), int(numa_node), C.byref(h)))
        return cls._adopt(shape, h, n_slots)

    @property
    def numa_node(self) -> int:
        """NUMA node backing the first page (-1: unknown / device pool)."""
        return lib.tsb_pool_numa_node(self._h)

    # ---- peer-HBM tier: the same slot layout resident in GPU memory ----
    @classmethod
    def _adopt(cls, shape: KVShape, h, n_slots: int, keepalive=None) -> "ChunkPool":
        self = cls.__new__(cls)
        self.shape, self._h, self.n_slots = shape, h, n_slots
        self.chunk_bytes = lib.tsb_pool_chunk_bytes(h)
        self._keepalive = keepalive
        return self

    @classmethod
    def create_device(cls, shape: KVShape, n_slots: int, device: int = 0) -> "ChunkPool":
        """HBM chunk pool on `device` (tsb_pool_create_device); export it with ipc_handle()."""
        h = C.c_void_p()
        check(lib.tsb_pool_create_device(int(device), C.byref(shape.struct()), int(n_slots), C.byref(h)))
        return cls._adopt(shape, h, n_slots)

    @classmethod
    def wrap_device(cls, shape: KVShape, tensor: torch.Tensor, n_slots: Optional[int] = None) -> "ChunkPool":
        """A CUDA tensor (kept alive by the pool) as the chunk pool (tsb_pool_wrap_device)."""
        n_slots = tensor.numel() * tensor.element_size() // shape.chunk_bytes if n_slots is None else n_slots
        h = C.c_void_p()
        check(lib.tsb_pool_wrap_device(tensor.device.index, C.byref(shape.struct()), tensor.data_ptr(),
                                       int(n_slots), C.byref(h)))
        return cls._adopt(shape, h, n_slots, keepalive=tensor)

    @classmethod
    def open_ipc(cls, shape: KVShape, handle: bytes, n_slots: int, owner_device: int = -1) -> "ChunkPool":
        """Map another process's create_device pool (cudaIpcOpenMemHandle, lazy peer access)."""
        if len(handle) != 64:
            raise ValueError("an IPC pool handle is 64 bytes")
        h = C.c_void_p()
        check(lib.tsb_pool_open_ipc(C.byref(shape.struct()), handle, int(owner_device), int(n_slots), C.byref(h)))
        return cls._adopt(shape, h, n_slots)

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(64)
        check(lib.tsb_pool_ipc_handle(self._h, buf))
        return buf.raw

    @property
    def on_device(self) -> bool:
        return lib.tsb_pool_location_of(self._h) == capi.POOL_DEVICE

    @property
    def device(self) -> int:
        return lib.tsb_pool_device(self._h)

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) and lib is not None:  # lib is None during interpreter exit
            lib.tsb_pool_destroy(self._h)
            self._h = None

    __del__ = close

    def slot_ptr(self, slot: int) -> int:
        """Host address of a slot (device address for a device pool)."""
        return lib.tsb_pool_slot_ptr(self._h, int(slot))

    def slot_view(self, slot: int, count: int = 1) -> np.ndarray:
        """Writable uint8 numpy view of `count` slots (host pools only)."""
        if self.on_device:
            raise TypeError("slot_view: the pool is in device memory")
        buf = (C.c_uint8 * (self.chunk_bytes * count)).from_address(self.slot_ptr(slot))
        return np.frombuffer(buf, dtype=np.uint8)

    def fill_synthetic(self, seed: int, first: int = 0, n: Optional[int] = None, stream=None):
        n = self.n_slots - first if n is None else n
        check(lib.tsb_pool_fill_synthetic(self._h, int(seed), int(first), int(n), _stream(stream)))


class PagedKVCache:
    """L1 tier: paged HBM arena + block_table, allocated with TierLedger semantics.

    request()/release_request() mirror TierLedger::request/release (engine.cpp:22-49) with
    capacity = num_pages * page_bytes; each granted chunk gets pages_per_chunk pages from a FIFO
    free list, written into the request's block_table row."""

    def __init__(self, shape: KVShape, num_pages: int, max_rows: int, max_chunks: int, device: int = 0,
                 arena: Optional[torch.Tensor] = None, layout: int = 0):
        self.shape = shape
        self.device = device
        self.num_pages = num_pages
        layer_bytes = 2 * num_pages * shape.page_tokens * shape.heads_local * shape.head_dim * shape.dtype_bytes
        if arena is None:
            arena = torch.empty(shape.layers * layer_bytes, dtype=torch.uint8, device=torch.device("cuda", device))
        if arena.numel() < shape.layers * layer_bytes or not arena.is_cuda:
            raise ValueError("arena must be a CUDA uint8 tensor of layers*2*num_pages*page*heads*dim*dtype bytes")
        self.arena = arena
        self.layer_bytes = layer_bytes
        h = C.c_void_p()
        check(lib.tsb_l1_create(device, C.byref(shape.struct()), int(num_pages), int(max_rows), int(max_chunks),
                                arena.data_ptr(), C.byref(h)))
        self._h = h
        self.max_rows, self.max_chunks = max_rows, max_chunks
        self.stride = lib.tsb_l1_block_table_stride(h)
        self.page_bytes = lib.tsb_l1_page_bytes(h)
        if layout != LAYOUT_FLASH_ATTN:
            check(lib.tsb_l1_set_layout(h, int(layout)))
        self.layout = layout

    @property
    def ce_group_bytes(self) -> int:
        """Cap on one CE staging group (0: half of the staging ring; tsb_l1_set_ce_group_bytes)."""
        return int(lib.tsb_l1_ce_group_bytes(self.handle))

    @ce_group_bytes.setter
    def ce_group_bytes(self, nbytes: int):
        check(lib.tsb_l1_set_ce_group_bytes(self.handle, int(nbytes)))

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) and lib is not None:  # lib is None during interpreter exit
            lib.tsb_l1_destroy(self._h)
            self._h = None

    __del__ = close

    def tier(self) -> Tier:
        return Tier.L1

    def request(self, request_id: int, block_index: int, nbytes: int):
        g, row = C.c_int(), C.c_int32()
        check(lib.tsb_l1_request(self._h, int(request_id), int(block_index), int(nbytes), C.byref(g), C.byref(row)))
        return bool(g.value), row.value

    def release_request(self, request_id: int):
        cap = max(64, self.deferred_count())
        out = (capi.Grant * cap)()
        n = C.c_int64()
        check(lib.tsb_l1_release_request(self._h, int(request_id), out, cap, C.byref(n)))
        return [(out[i].request_id, out[i].block_index, out[i].bt_row, out[i].bytes) for i in range(min(n.value, cap))]

    def capacity(self) -> int:
        return lib.tsb_l1_capacity(self._h)

    def reserved(self) -> int:
        return lib.tsb_l1_reserved(self._h)

    def deferred_count(self) -> int:
        return lib.tsb_l1_deferred(self._h)

    def free_pages(self) -> int:
        return lib.tsb_l1_free_pages(self._h)

    def block_table(self) -> np.ndarray:
        """Host (pinned) mirror [max_rows, max_chunks*pages_per_chunk] int32 (a view)."""
        n = self.max_rows * self.stride
        buf = (C.c_int32 * n).from_address(lib.tsb_l1_block_table_host(self._h))
        return np.frombuffer(buf, dtype=np.int32).reshape(self.max_rows, self.stride)

    def sync_block_table(self, stream=None):
        check(lib.tsb_l1_sync_block_table(self._h, _stream(stream)))

    def block_table_device(self) -> torch.Tensor:
        """The device block table [max_rows, stride] int32 (a view; rows are uploaded by
        sync_block_table / the load stage ahead of the ingest that reads them).  The view aliases
        memory the L1 owns: keep this PagedKVCache alive while it is used."""
        ptr = lib.tsb_l1_block_table_device(self._h)

        class _View:  # __cuda_array_interface__ over memory the L1 object owns
            __cuda_array_interface__ = {"shape": (self.max_rows, self.stride), "typestr": "<i4",
                                        "data": (ptr, False), "version": 3, "strides": None}

        return torch.as_tensor(_View(), device=torch.device("cuda", self.device))

    def layer(self, layer: int, dtype=torch.bfloat16) -> torch.Tensor:
        """One layer in the consumer's layout: flash-attn [2, pages, P, H_local, D]; FlashInfer NHD
        [pages, 2, P, H_local, D]; FlashInfer HND [pages, 2, H_local, P, D]."""
        s = self.shape
        t = self.arena[layer * self.layer_bytes:(layer + 1) * self.layer_bytes].view(dtype)
        if self.layout == LAYOUT_FLASHINFER_NHD:
            return t.view(self.num_pages, 2, s.page_tokens, s.heads_local, s.head_dim)
        if self.layout == LAYOUT_FLASHINFER_HND:
            return t.view(self.num_pages, 2, s.heads_local, s.page_tokens, s.head_dim)
        return t.view(2, self.num_pages, s.page_tokens, s.heads_local, s.head_dim)


def items_numpy(src_slot, bt_row, chunk_index) -> np.ndarray:
    dt = np.dtype([("src_slot", np.int64), ("bt_row", np.int32), ("chunk_index", np.int32)])
    a = np.empty(len(src_slot), dtype=dt)
    a["src_slot"], a["bt_row"], a["chunk_index"] = src_slot, bt_row, chunk_index
    return a


def _items_ptr(items):
    if isinstance(items, np.ndarray):
        return C.cast(items.ctypes.data, C.POINTER(capi.IngestItem)), len(items)
    return items, len(items)


def _events(layer_events, n_layers):
    if layer_events is None:
        return None
    assert len(layer_events) == n_layers, "one event (or None) per layer of the range"
    arr = (C.c_void_p * n_layers)()
    for i, e in enumerate(layer_events):
        if e is not None and not e.cuda_event:
            e.record()  # torch creates the cudaEvent_t lazily on first record
        arr[i] = e.cuda_event if e is not None else None
    return arr


def ingest(l1: PagedKVCache, pool: ChunkPool, items, layer_lo: int = 0, layer_hi: Optional[int] = None,
           mode: int = AUTO, stream=None, layer_events: Optional[Sequence] = None):
    """tsb_ingest: moves every (item, layer in [layer_lo, layer_hi)) L2 -> L1 (async on `stream`);
    layer_events[k] (torch.cuda.Event or None) is recorded once layer layer_lo+k is resident."""
    layer_hi = l1.shape.layers if layer_hi is None else layer_hi
    ptr, n = _items_ptr(items)
    check(lib.tsb_ingest(l1.handle, pool.handle, ptr, n, layer_lo, layer_hi, int(mode), _stream(stream),
                         _events(layer_events, layer_hi - layer_lo)))


def ingest_tiered(l1: PagedKVCache, pool: Optional[ChunkPool], hbm_pool: Optional[ChunkPool], items, layer_lo: int = 0,
                  layer_hi: Optional[int] = None, mode: int = AUTO, stream=None,
                  layer_events: Optional[Sequence] = None):
    """tsb_ingest_tiered: items with src_slot < 0 come from slot ~src_slot of hbm_pool (the HBM tier,
    K1 at HBM / NVLink speed), the rest from pool; the fences cover both."""
    layer_hi = l1.shape.layers if layer_hi is None else layer_hi
    ptr, n = _items_ptr(items)
    check(lib.tsb_ingest_tiered(l1.handle, pool.handle if pool is not None else None,
                                hbm_pool.handle if hbm_pool is not None else None, ptr, n,
                                layer_lo, layer_hi, int(mode), _stream(stream),
                                _events(layer_events, layer_hi - layer_lo)))


def ingest_device(l1: PagedKVCache, pool: ChunkPool, items_dev: torch.Tensor, n_items: int, layer_lo: int = 0,
                  layer_hi: Optional[int] = None, mode: int = AUTO, stream=None, layer_events=None):
    layer_hi = l1.shape.layers if layer_hi is None else layer_hi
    check(lib.tsb_ingest_device(l1.handle, pool.handle, items_dev.data_ptr(), int(n_items), layer_lo, layer_hi,
                                int(mode), _stream(stream), _events(layer_events, layer_hi - layer_lo)))


def verify_synthetic(l1: PagedKVCache, pool: ChunkPool, items, seed: int, layer_lo: int = 0,
                     layer_hi: Optional[int] = None, stream=None) -> int:
    layer_hi = l1.shape.layers if layer_hi is None else layer_hi
    ptr, n = _items_ptr(items)
    out = C.c_uint64()
    check(lib.tsb_l1_verify_synthetic(l1.handle, ptr, n, layer_lo, layer_hi, int(seed), pool.chunk_bytes,
                                      _stream(stream), C.byref(out)))
    return out.value


def set_grid(zerocopy_ctas: int = 0, bulk_ctas: int = 0, scatter_ctas: int = 0):
    check(lib.tsb_ingest_set_grid(zerocopy_ctas, bulk_ctas, scatter_ctas))


def enable_peer_access(device: int, peer: int):
    check(lib.tsb_enable_peer_access(int(device), int(peer)))


def resolve_mode(l1: PagedKVCache, pool: ChunkPool, items=None, mode: int = AUTO) -> int:
    """The kernel path tsb_ingest takes for these items (AUTO resolved; items=None: device items)."""
    ptr, n = _items_ptr(items) if items is not None else (None, 0)
    out = C.c_int()
    check(lib.tsb_ingest_resolve_mode(l1.handle, pool.handle, ptr, n, int(mode), C.byref(out)))
    return out.value


def set_ce(variant: int = 1, staging_bytes: int = 0):
    """CE copy strategy: 0 per-item memcpy, 1 2D copy per consecutive-slot run (default)."""
    check(lib.tsb_ingest_set_ce(variant, staging_bytes))
