"""Probe: per-call wall time of the host-buffer scorer entry (tsb_score_queue), 100K queue."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tools"))
import numpy as np
from bench_queue import loogle_queue
from paper_2603_21257_b200 import tiersim as t
from paper_2603_21257_b200.scorer import BatchScorer
import os
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
q = loogle_queue(100_000, 0)
cfg = t.ClusterConfig(); m = t.cost_models_from_config(cfg)
sc = BatchScorer(0)
outs = [np.empty(100_000) for _ in range(3)] + [np.empty(100_000, np.int64)]
for k in range(12):
    t0 = time.perf_counter()
    sc.score(q, t.PolicyKind.Lstf, m, cfg)
    t1 = time.perf_counter()
    print(f"call {k}: {1e6*(t1-t0):.0f} us")
import torch
s = torch.cuda.Stream()
for k in range(4):
    t0 = time.perf_counter()
    sc.score(q, t.PolicyKind.Lstf, m, cfg, stream=s)
    print(f"explicit stream call {k}: {1e6*(time.perf_counter()-t0):.0f} us")
n = 6_500_000
h = torch.empty(n, dtype=torch.uint8).pin_memory(); d = torch.empty(n, dtype=torch.uint8, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for k in range(4):
    h.fill_(k)
    a.record(); d.copy_(h, non_blocking=True); b.record(); b.synchronize()
    print(f"torch pinned h2d in-process: {a.elapsed_time(b)*1e3:.0f} us")
from paper_2603_21257_b200 import ingest
p = ingest.ChunkPool(ingest.KVShape(layers=1, kv_heads=8, head_dim=128), 13)  # 6.8 MB, cudaHostAlloc portable|mapped
hv = p.slot_view(0, 13)
ht = torch.from_numpy(hv)
for k in range(3):
    hv[:] = k
    a.record(); d[:n].copy_(ht[:n], non_blocking=True); b.record(); b.synchronize()
    print(f"libtsb pool pinned h2d in-process: {a.elapsed_time(b)*1e3:.0f} us")
