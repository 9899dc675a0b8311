"""Sweep K2 (paged scatter from HBM staging) implementations and grids; device-timed."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import measure_k2  # noqa: E402
from paper_2603_21257_b200 import ingest  # noqa: E402
from paper_2603_21257_b200._capi import lib  # noqa: E402

shape = ingest.QWEN25_32B
l1 = ingest.PagedKVCache(shape, 8192, max_rows=2, max_chunks=512)
for impl, grids in ((0, [148 * 4, 148 * 8, 148 * 16, 148 * 32]), (1, [0])):
    for g in grids:
        lib.tsb_ingest_set_scatter(impl, g)
        for n_items in (128, 460):
            nbytes, secs = measure_k2(torch, l1, shape, n_items=n_items, reps=30)
            print(json.dumps(dict(impl=["sm_ldg", "tma_k1b"][impl], ctas=g, items=n_items, us=secs * 1e6,
                                  GBps=nbytes / secs / 1e9, hbm_frac=nbytes / secs / 1e9 / 6450.6)), flush=True)
lib.tsb_ingest_set_scatter(0, 0)
