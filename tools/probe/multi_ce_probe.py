"""Is 55.6 GB/s a single-copy-engine limit or the link?  Concurrent H2D copies on N streams."""
import json

import torch

n = 1 << 30
for k in (1, 2, 3, 4):
    hs = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(k)]
    ds = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(k)]
    ss = [torch.cuda.Stream() for _ in range(k)]
    best = 1e9
    for rep in range(4):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(k):
            ss[i].wait_event(a)
            with torch.cuda.stream(ss[i]):
                ds[i].copy_(hs[i], non_blocking=True)
        for i in range(k):
            torch.cuda.current_stream().wait_stream(ss[i])
        b.record()
        b.synchronize()
        if rep:
            best = min(best, a.elapsed_time(b) * 1e-3)
    print(json.dumps({"streams": k, "aggregate_GBps": k * n / best / 1e9}), flush=True)
    del hs, ds
