"""Probe: host cost of one PagedPrefill hook call (one layer of one request's prefill), with the
GPU otherwise idle and with the compute stream already holding work -- is the consumer's enqueue
host-bound?  Probe only; not product code."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2603_21257_b200 import ingest  # noqa: E402
from paper_2603_21257_b200 import tiersim as t  # noqa: E402
from paper_2603_21257_b200.consumer import PagedPrefill  # noqa: E402


def main():
    shape = ingest.LLAMA31_8B
    n, ctx, hit = 4, 32768, 0.97
    nb = int(np.floor(ctx * hit / 256))
    pool = ingest.ChunkPool(shape, nb)
    pool.fill_synthetic(1)
    l1 = ingest.PagedKVCache(shape, n * nb * 16 + 16, max_rows=n + 1, max_chunks=nb)
    q = t.QueueArrays(n, id=np.arange(n), arrival=np.zeros(n), context_tokens=np.full(n, ctx),
                      query_tokens=np.full(n, 28), cache_hit_ratio=np.full(n, hit), flags=np.zeros(n, np.uint8))
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(32, 8, 128, 2))
    rows = []
    for i in range(n):
        for c in range(nb):
            rows.append(l1.request(i, c, shape.page_bytes * 16)[1])
    l1.sync_block_table()
    row_of = [rows[i * nb] for i in range(n)]
    cons = PagedPrefill(l1, q, cfg)
    s = torch.cuda.Stream(priority=0)
    for i in range(2):  # warm-up (cuBLAS / FlashInfer JIT)
        for layer in range(32):
            cons(i, row_of[i], layer, s.cuda_stream)
    torch.cuda.synchronize()
    for case in ("idle", "backlog"):
        i = 2 if case == "idle" else 3
        if case == "backlog":  # ~1 s of GEMMs already queued on the compute stream
            with torch.cuda.stream(s):
                x = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
                for _ in range(800):
                    x = x @ x * 1e-4
        per = []
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for layer in range(32):
            t0 = time.perf_counter()
            cons(i, row_of[i], layer, s.cuda_stream)
            per.append(time.perf_counter() - t0)
        b.record(s)
        host_total = sum(per)
        b.synchronize()
        print(json.dumps({"probe": "hook_cost", "case": case, "host_ms_per_layer_mean": 1e3 * host_total / 32,
                          "host_ms_layer0": 1e3 * per[0], "host_ms_max": 1e3 * max(per),
                          "gpu_ms_request": a.elapsed_time(b) if case == "idle" else None}), flush=True)


if __name__ == "__main__":
    main()
