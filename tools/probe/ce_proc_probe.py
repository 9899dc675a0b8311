"""Copy-engine H2D rate of one process over a fixed window (run several at once to see whether
separate processes / contexts share the link better than streams of one process).
    python tools/probe/ce_proc_probe.py [seconds] [streams]"""
import json
import os
import sys
import time

import torch

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1
n = 1 << 30
hs = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(k)]
ds = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(k)]
ss = [torch.cuda.Stream() for _ in range(k)]
for i in range(k):
    ds[i].copy_(hs[i])
torch.cuda.synchronize()
t0 = time.time()
moved = 0
while time.time() - t0 < secs:
    for i in range(k):
        with torch.cuda.stream(ss[i]):
            ds[i].copy_(hs[i], non_blocking=True)
    torch.cuda.synchronize()
    moved += k * n
dt = time.time() - t0
print(json.dumps({"pid": os.getpid(), "streams": k, "env_copy_conn": os.environ.get("CUDA_DEVICE_MAX_COPY_CONNECTIONS"),
                  "GBps": moved / dt / 1e9, "t0": t0, "t1": t0 + dt}), flush=True)
