"""Peer-HBM tier: ingest from a chunk pool resident in GPU memory.

On the one-GPU box the pool is local HBM, so the copy is HBM -> HBM (read + write) and the
roofline is the measured HBM bandwidth; with a peer GPU the same kernels read over NVLink 5 and
the bound becomes the per-direction NVLink rate.  One JSON line per (workload, mode, tp).
Device-timed with CUDA events on the launching stream, best of `reps` after warm-up; inputs are
larger than L2 (4.3-10.7 GB per call).
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_21257_b200 import ingest  # noqa: E402
from paper_2603_21257_b200._capi import lib  # noqa: E402


def hbm_peak():
    from bench import measured_peaks  # noqa: E402

    return measured_peaks()[0]


def run(shape, n_chunks, mode, reps, seed=3, layout=0):
    pool = ingest.ChunkPool.create_device(shape, n_chunks)
    pool.fill_synthetic(seed)
    ppc = shape.pages_per_chunk
    l1 = ingest.PagedKVCache(shape, n_chunks * ppc, max_rows=1, max_chunks=n_chunks, layout=layout)
    for c in range(n_chunks):
        assert l1.request(1, c, shape.page_bytes * ppc)[0]
    l1.sync_block_table()
    items = ingest.items_numpy(np.random.default_rng(seed).permutation(n_chunks), np.zeros(n_chunks, np.int32),
                               np.arange(n_chunks, dtype=np.int32))
    dev_items = torch.from_numpy(items.view(np.uint8).copy()).cuda()
    s = torch.cuda.Stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    with torch.cuda.stream(s):
        for r in range(reps + 2):
            a.record(s)
            ingest.ingest_device(l1, pool, dev_items, n_chunks, mode=mode, stream=s)
            b.record(s)
            b.synchronize()
            if r >= 2:
                best = min(best, a.elapsed_time(b) * 1e-3)
    bad = ingest.verify_synthetic(l1, pool, items, seed=seed)
    payload = n_chunks * shape.local_chunk_bytes
    l1.close()
    pool.close()
    return payload, best, bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    peak = hbm_peak()
    cases = [("llama8b32k", ingest.LLAMA31_8B, 128, (1, 0)),
             ("qwen32b_64chunks", ingest.QWEN25_32B, 64, (1, 0)),
             ("llama70b32k_tp8", ingest.LLAMA3_70B, 128, (8, 0)),
             ("llama70b32k_tp4", ingest.LLAMA3_70B, 128, (4, 1)),
             ("llama70b32k_tp2", ingest.LLAMA3_70B, 128, (2, 0))]
    for name, shape, n, tp in cases:
        shape = shape.with_rank(*tp)
        for layout in ("flash_attn", "flashinfer_hnd"):
          for mname in ("zerocopy", "bulk"):
            payload, secs, bad = run(shape, n, ingest.MODES[mname], args.reps, layout=ingest.LAYOUTS[layout])
            gbs = payload / secs / 1e9
            print(json.dumps(dict(workload=name, source="device_pool_local_hbm", mode=mname, tp=tp[0], layout=layout,
                                  payload_bytes=payload, ms=secs * 1e3, payload_GBps=round(gbs, 1),
                                  hbm_GBps=round(2 * gbs, 1), hbm_peak_GBps=peak,
                                  frac=round(2 * gbs / peak, 4), verify_mismatches=int(bad))), flush=True)
    lib.tsb_ingest_set_grid(0, 0, 0)


if __name__ == "__main__":
    main()
