"""Probe: does a concurrent prefill slow the copy-engine ingest on the device, or is it the host?

Ingest of 64 Llama-3.1-8B chunks (4.3 GB) with CE-direct and CE+K2, alone and while a prefill
workload runs on another stream: bf16 GEMMs only, FlashInfer paged prefill only (reading the same
arena), and both -- each queued as ~2 s of work BEFORE the ingest starts, so no host time is spent
enqueueing during the ingest.  Prints one JSON line per case.  Probe only; not product code.
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2603_21257_b200 import ingest  # noqa: E402


def main():
    import flashinfer

    shape = ingest.LLAMA31_8B
    n = 64
    pool = ingest.ChunkPool(shape, n)
    pool.fill_synthetic(1)
    l1 = ingest.PagedKVCache(shape, 2 * n * 16, max_rows=2, max_chunks=n)
    cb = shape.page_bytes * 16
    rows = [l1.request(1, c, cb)[1] for c in range(n)]
    rows2 = [l1.request(2, c, cb)[1] for c in range(n)]
    l1.sync_block_table()
    items = ingest.items_numpy(np.arange(n), [rows[0]] * n, np.arange(n))
    dev = torch.device("cuda")
    ingest.ingest(l1, pool, ingest.items_numpy(np.arange(n), [rows2[0]] * n, np.arange(n)))  # KV for attention
    torch.cuda.synchronize()
    # prefill pieces: 8K new tokens over a 16K-token cached prefix (row 2), Llama-8B layer GEMMs
    ct, hid, inter = 8192, 4096, 14336
    x = torch.randn(ct, hid, device=dev, dtype=torch.bfloat16)
    w1 = torch.randn(hid, 2 * inter, device=dev, dtype=torch.bfloat16) * 0.01
    w2 = torch.randn(inter, hid, device=dev, dtype=torch.bfloat16) * 0.01
    ws = torch.empty(128 << 20, dtype=torch.uint8, device=dev)
    wr = flashinfer.BatchPrefillWithPagedKVCacheWrapper(ws, "NHD")
    pages = torch.from_numpy(np.ascontiguousarray(l1.block_table()[rows2[0], : n * 16])).to(dev)
    i32 = dict(dtype=torch.int32)
    wr.plan(torch.tensor([0, ct], **i32), torch.tensor([0, n * 16], **i32), pages, torch.tensor([16], **i32),
            32, 8, 128, 16, causal=False, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
    q = torch.randn(ct, 32, 128, device=dev, dtype=torch.bfloat16)
    kv = l1.layer(3)
    comp = torch.cuda.Stream(priority=0)
    ing = torch.cuda.Stream(priority=-1)

    def gemms(k):
        for _ in range(k):
            h = x @ w1
            x.copy_(h[:, :inter] @ w2)

    def attn(k):
        for _ in range(k):
            wr.run(q, (kv[0], kv[1]))

    def ingest_once(mode, fenced):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        evs = [torch.cuda.Event() for _ in range(shape.layers)] if fenced else None
        a.record(ing)
        ingest.ingest(l1, pool, items, mode=mode, stream=ing, layer_events=evs)
        b.record(ing)
        b.synchronize()
        return n * shape.chunk_bytes / (a.elapsed_time(b) * 1e-3) / 1e9

    for mode_name, fenced in (("ce_direct", False), ("ce_direct", True), ("ce", False), ("ce", True)):
        mode = ingest.MODES[mode_name]
        ingest_once(mode, fenced)
        for load in ("none", "gemm", "attention", "both"):
            torch.cuda.synchronize()
            with torch.cuda.stream(comp):
                if load in ("gemm", "both"):
                    gemms(60)
                if load in ("attention", "both"):
                    attn(40)
            gbs = ingest_once(mode, fenced)
            busy = not comp.query()
            torch.cuda.synchronize()
            print(json.dumps({"probe": "ingest_under_prefill", "mode": mode_name, "per_layer_fences": fenced,
                              "concurrent": load, "GBps": round(gbs, 2),
                              "prefill_still_running_at_end": busy}), flush=True)


if __name__ == "__main__":
    main()
