"""A real layer-pipelined prefill consumer of the ingested pages.

The reference's compute stage is a duration, compute_base + per_token * n (engine.cpp:210-212,
448-473).  PagedPrefill is an actual per-layer prefill of a Llama-3.1-8B-sized decoder layer,
enqueued on the load stage's compute stream through its prefill hook (tsb_stage_set_prefill_hook):
for layer l of a request, after the stage made the stream wait for that layer's ingest fence,

  qkv = x @ W_qkv                          (bf16 GEMM, cuBLAS)
  o   = paged attention of q over the request's cached pages of layer l, read in place from the
        L1 arena through our block table (FlashInfer BatchPrefillWithPagedKVCacheWrapper)
  h   = o @ W_o;  y = (silu(h @ W_gate) * (h @ W_up)) @ W_down   (MLP, token-blocked)

so prefill of layer l overlaps ingest of layers > l, and it reads the very pages K2 wrote: HBM
and SM interference are real.  Weights are random and shared by all layers (the same FLOPs per
layer as distinct weights, a 32x smaller footprint); the new tokens attend to the cached prefix
only (their own K/V are not appended), which keeps the attention FLOPs of the cached part exact.
"""
from __future__ import annotations

import time
from typing import Optional

import numpy as np
import torch

from .ingest import LAYOUT_FLASH_ATTN, LAYOUT_FLASHINFER_HND, PagedKVCache
from .tiersim import ClusterConfig, QueueArrays


class PagedPrefill:
    def __init__(self, l1: PagedKVCache, queue: QueueArrays, config: ClusterConfig, hidden: int = 4096,
                 q_heads: int = 32, intermediate: int = 14336, token_block: int = 8192, wrappers: int = 0,
                 seed: int = 0, preplan: Optional[bool] = None):
        import flashinfer

        self.l1, self.queue, self.config = l1, queue, config
        s = l1.shape
        self.D, self.Hkv, self.Hq = s.head_dim, s.heads_local, q_heads
        dev = torch.device("cuda", l1.device)
        g = torch.Generator(device=dev).manual_seed(seed)
        bf = torch.bfloat16
        w = lambda i, o: (torch.randn(i, o, device=dev, dtype=bf, generator=g) * (i ** -0.5)).to(bf)
        self.w_qkv = w(hidden, (q_heads + 2 * self.Hkv) * self.D)
        self.w_o = w(q_heads * self.D, hidden)
        self.w_gu = w(hidden, 2 * intermediate)
        self.w_down = w(intermediate, hidden)
        self.token_block = token_block
        # compute tokens per request (types.cpp:81-83) and the activations of the longest one
        bpt = s.chunk_tokens
        self.ct = [int(queue.context_tokens[i] + queue.query_tokens[i]
                       - np.floor(queue.context_tokens[i] * queue.cache_hit_ratio[i] / bpt) * bpt)
                   for i in range(queue.n)]
        self.nb = [int(np.floor(queue.context_tokens[i] * queue.cache_hit_ratio[i] / bpt)) for i in range(queue.n)]
        self.x = torch.randn(max(self.ct + [1]), hidden, device=dev, dtype=bf, generator=g) * 0.5
        self.q_buf = torch.empty(max(self.ct + [1]), q_heads, self.D, device=dev, dtype=bf)
        self.o_buf = torch.empty_like(self.q_buf)
        layout = "HND" if l1.layout == LAYOUT_FLASHINFER_HND else "NHD"
        self.kv_tuple = l1.layout == LAYOUT_FLASH_ATTN
        # A wrapper per request up to 128 (each holds one request's plan: 8 MiB of device and of
        # pinned metadata); beyond that a ring whose wrappers are re-planned once the prefill that
        # used them has finished.  The 128 MiB split-k float workspace is shared: every run is
        # serialized on the one compute stream.
        wrappers = wrappers or max(2, min(128, queue.n))
        self.float_ws = torch.empty(128 << 20, dtype=torch.uint8, device=dev)
        self.wrappers = [flashinfer.BatchPrefillWithPagedKVCacheWrapper(self.float_ws, layout) for _ in range(wrappers)]
        self.done = [None] * wrappers
        # per wrapper: pinned staging of the page list (copied async) + host indptr tensors; all
        # reused only after the prefill that used them has finished, so nothing here syncs the
        # compute stream (the stage's host loop must keep the link busy meanwhile)
        max_pages = max(self.nb + [1]) * s.pages_per_chunk
        self.pin_pages = [torch.empty(max_pages, dtype=torch.int32, pin_memory=True) for _ in range(wrappers)]
        self.dev_pages = [torch.empty(max_pages, dtype=torch.int32, device=dev) for _ in range(wrappers)]
        self.host_meta = [(torch.zeros(2, dtype=torch.int32, pin_memory=True),
                           torch.zeros(2, dtype=torch.int32, pin_memory=True),
                           torch.zeros(1, dtype=torch.int32, pin_memory=True)) for _ in range(wrappers)]
        self.slot_of = {}
        self.next = 0
        # With a wrapper per request the attention is planned here, before any ingest: a plan
        # uploads its metadata with small host-to-device copies, and issued during the run those
        # copies queue behind the bulk KV copies on the copy engine -- the request's prefill could
        # not start before its last layer landed, defeating the per-layer fences
        # (repo:profiles/r02_layer_pipelining.jsonl).  The page list is then a device buffer that
        # layer 0 fills from the device block table with a kernel, no copy engine involved.
        self.bt_dev = l1.block_table_device()
        self.preplanned = queue.n <= wrappers if preplan is None else (preplan and queue.n <= wrappers)
        if self.preplanned:
            for i in range(queue.n):
                if self.nb[i] > 0:
                    self._plan_static(i, i)
            torch.cuda.synchronize(dev)
        self.flops = 0.0
        self.calls = 0
        self.host_s = 0.0       # host time spent inside the hook (enqueueing)
        self.host_max_s = 0.0
        self.plan_s = 0.0

    def flops_per_request(self, i: int) -> float:
        """GEMM + attention FLOPs of one request's prefill across all layers."""
        ct, kv = self.ct[i], self.nb[i] * self.l1.shape.chunk_tokens
        hidden, inter = self.w_qkv.shape[0], self.w_down.shape[0]
        gemm = 2 * ct * (hidden * self.w_qkv.shape[1] + self.w_o.shape[0] * hidden + hidden * 2 * inter + inter * hidden)
        attn = 4 * ct * kv * self.Hq * self.D
        return float(self.l1.shape.layers * (gemm + attn))

    def _plan_static(self, q_index: int, k: int):
        """Plan request q_index on wrapper k with dev_pages[k] as its page list (filled later)."""
        n_pages = self.nb[q_index] * self.l1.shape.pages_per_chunk
        qo, kvp, last = self.host_meta[k]
        qo[1], kvp[1], last[0] = self.ct[q_index], n_pages, self.l1.shape.page_tokens
        self.wrappers[k].plan(qo, kvp, self.dev_pages[k][:n_pages], last, self.Hq, self.Hkv, self.D,
                              self.l1.shape.page_tokens, causal=False, q_data_type=torch.bfloat16,
                              kv_data_type=torch.bfloat16)
        self.slot_of[q_index] = k

    def _plan(self, q_index: int, bt_row: int):
        k = self.next % len(self.wrappers)
        self.next += 1
        if self.done[k] is not None:
            self.done[k].synchronize()  # the prefill that last used this wrapper has finished
        n_pages = self.nb[q_index] * self.l1.shape.pages_per_chunk
        pin, dpages = self.pin_pages[k], self.dev_pages[k]
        pin[:n_pages].copy_(torch.from_numpy(np.ascontiguousarray(self.l1.block_table()[bt_row, :n_pages])))
        dpages[:n_pages].copy_(pin[:n_pages], non_blocking=True)
        qo, kvp, last = self.host_meta[k]
        qo[1], kvp[1], last[0] = self.ct[q_index], n_pages, self.l1.shape.page_tokens
        self.wrappers[k].plan(qo, kvp, dpages[:n_pages], last, self.Hq, self.Hkv, self.D, self.l1.shape.page_tokens,
                              causal=False, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
        self.slot_of[q_index] = k

    def __call__(self, q_index: int, bt_row: int, layer: int, stream_ptr: int):
        """The stage's prefill hook: enqueue layer `layer` of request q_index on `stream_ptr`."""
        t0 = time.perf_counter()
        try:
            self._enqueue(q_index, bt_row, layer, stream_ptr)
        finally:
            dt = time.perf_counter() - t0
            self.host_s += dt
            self.host_max_s = max(self.host_max_s, dt)

    def _enqueue(self, q_index: int, bt_row: int, layer: int, stream_ptr: int):
        stream = torch.cuda.ExternalStream(stream_ptr, device=self.x.device)
        with torch.cuda.stream(stream):
            ct = self.ct[q_index]
            if ct == 0:
                return
            if layer == 0 and self.nb[q_index] > 0:
                t0 = time.perf_counter()
                if self.preplanned:  # the request's pages, device block table -> its page list
                    n_pages = self.nb[q_index] * self.l1.shape.pages_per_chunk
                    k = self.slot_of[q_index]
                    torch.add(self.bt_dev[bt_row, :n_pages], 0, out=self.dev_pages[k][:n_pages])
                else:
                    self._plan(q_index, bt_row)
                self.plan_s += time.perf_counter() - t0
            x = self.x[:ct]
            qkv = x @ self.w_qkv
            q = self.q_buf[:ct]
            q.copy_(qkv[:, : self.Hq * self.D].view(ct, self.Hq, self.D))
            if self.nb[q_index] > 0:
                kv = self.l1.layer(layer)
                wr = self.wrappers[self.slot_of[q_index]]
                o = wr.run(q, (kv[0], kv[1]) if self.kv_tuple else kv, out=self.o_buf[:ct])
            else:
                o = q
            h = o.reshape(ct, -1) @ self.w_o
            inter = self.w_down.shape[0]
            for t0 in range(0, ct, self.token_block):  # token-blocked MLP: bounded activations
                hb = h[t0:t0 + self.token_block]
                gu = hb @ self.w_gu
                a = torch.nn.functional.silu(gu[:, :inter]) * gu[:, inter:]
                hb.copy_(a @ self.w_down)
            if layer == self.l1.shape.layers - 1 and self.nb[q_index] > 0 and not self.preplanned:
                ev = torch.cuda.Event()
                ev.record(stream)
                self.done[self.slot_of[q_index]] = ev
        self.calls += 1
        if layer == 0:
            self.flops += self.flops_per_request(q_index)
