#!/bin/bash
# Round 2: K1b ring size (bytes of segment buffers per CTA ring; CTAs per SM follow) over the
# (TSB_K1B_RING was a one-off switch in kernels.h, removed once 64 KiB rings for <= 8 KiB segments shipped)
# peer-tier shapes -- default 96 KiB vs 64 / 48 / 128 KiB.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for r in 98304 65536 49152 131072; do
  TSB_K1B_RING=$r timeout 600 python tools/bench_peer.py > gpurun_out/k1b_ring_${r}.jsonl 2>/dev/null; echo "ring $r rc=$?"
done
