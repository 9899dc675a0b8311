"""Where a small `value` step goes (configs[0], HBM-resident pool): the stage call vs its K1
launches vs the scorer round trip.  Probe only.   python tools/probe/stage_overhead_probe.py"""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2603_21257_b200 import ingest
from paper_2603_21257_b200.stage import LoadStage
from paper_2603_21257_b200.workloads import WORKLOADS
from paper_2603_21257_b200.tiersim import PolicyKind
from paper_2603_21257_b200.scorer import BatchScorer
from paper_2603_21257_b200 import tiersim as t
wl = WORKLOADS['llama8b32k']()
shape = wl.shape
dpool = ingest.ChunkPool.create_device(shape, wl.pool_slots); dpool.fill_synthetic(1)
l1 = ingest.PagedKVCache(shape, 4096, max_rows=4, max_chunks=128)
st = LoadStage(l1, dpool)
s = torch.cuda.current_stream()
def timeit(f, n=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record(s)
    for _ in range(n): f()
    b.record(s); b.synchronize()
    return a.elapsed_time(b) / n, (time.perf_counter() - t0) * 1e3 / n
print('stage.run', timeit(lambda: st.run(wl.queue, wl.slots, wl.config, policy=PolicyKind.Fifo)))
print('stage.run layer_events', timeit(lambda: st.run(wl.queue, wl.slots, wl.config, policy=PolicyKind.Fifo, layer_events=True)))
sc = BatchScorer(0)
cfg = wl.config; m = t.cost_models_from_config(cfg)
print('score n=1', timeit(lambda: sc.score(wl.queue, PolicyKind.Fifo, m, cfg)))
for c in range(128): l1.request(99, c, shape.page_bytes * 16)
l1.sync_block_table()
items = ingest.items_numpy(np.arange(128), [0] * 128, np.arange(128))
bt = l1.block_table(); row = int(np.where((bt >= 0).any(axis=1))[0][0])
items['bt_row'] = row
dev_items = torch.from_numpy(items.view(np.uint8).copy()).cuda()
print('K1 [0,L) one launch', timeit(lambda: ingest.ingest_device(l1, dpool, dev_items, 128, 0, shape.layers, mode=ingest.ZEROCOPY, stream=s)))
print('K1 [0,1)+[1,L)', timeit(lambda: (ingest.ingest_device(l1, dpool, dev_items, 128, 0, 1, mode=ingest.ZEROCOPY, stream=s), ingest.ingest_device(l1, dpool, dev_items, 128, 1, shape.layers, mode=ingest.ZEROCOPY, stream=s))))
print('tsb_ingest host items [0,L) with first/last fences', timeit(lambda: ingest.ingest(l1, dpool, items, layer_events=[torch.cuda.Event()] + [None]*(shape.layers-2) + [torch.cuda.Event()])))
