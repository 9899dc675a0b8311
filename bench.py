#!/usr/bin/env python3
"""Contract benchmark: KV ingest GB/s (L2 pinned host chunk pool -> L1 paged HBM) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload ...]

A step is one pass of the load stage over the batch: GPU scoring + pick order, TierLedger-
semantics page grants with FIFO deferral, block-table upload, ingest of every planned chunk, and
page release (tsb_stage_run, the public C-ABI call).  Default workload = BASELINE.json configs[1]
(Qwen2.5-32B KV, 16 x 128K @ 0.9 hit).  With N GPUs the KV heads are sharded TP-style: every rank
ingests its head slice of the same batch from its own NUMA-local pinned pool (strong scaling, no
data-path collective).  Without torchrun, --gpus N > 1 launches the N ranks itself.

  value    : the north-star hop, L2 pinned host pool -> L1 pages; payload bytes of all ranks / max
             over ranks of the CUDA-event time of the K timed stage passes (engine.cpp:206-207,
             427-446 made real)
  e2e      : the same K passes timed by the host wall clock around the public API calls
             (tsb_stage_run: queue + block-table uploads, results read back)
  roofline : the value arm's bound -- the host link, achieved per-GPU GB/s against the live
             copy-engine H2D peak of this box; K2 (the paged scatter that follows the copy
             engines, HBM-bound) is reported beside it with its ncu DRAM bytes (roofline_k2)
  hbm_tier : the same step with the pool held in HBM (the peer-HBM tier's K1 path), not the
             headline
  workloads: driver-visible lines for configs[0] (Llama-8B 32K), configs[2] (70B, rank 0 of a
             tp 1/2/4/8 head split on this GPU), configs[3] (mixed trace, K6 prefill), the real
             consumer's layer pipelining (f1) and configs[4] (100K-request scorer + hasher)
  cpu_baseline : the oracle's scatter_ref (port) on the host cores, bounded sample (rank 0, N=1)
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import socket
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "KV ingest GB/s per GPU and aggregate vs host-link/HBM roofline; TTFT load ms"
UNIT = "GB/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
GEN5_X16_GBS = 63.0        # PCIe Gen5 x16 per direction, theory

# BASELINE.json configs as plain numbers (the reference arm builds its sample from these without
# importing the product package; tests/test_bench_cpu.py checks they equal workloads.WORKLOADS).
SPECS = {
    "qwen16x128k": dict(name="qwen2.5-32b_16x128k_hit0.9", layers=64, kv_heads=8, head_dim=128, n_req=16,
                        ctx=131072, hit=0.9, query=28, n_docs=2),
    "llama8b32k": dict(name="llama3.1-8b_1x32k", layers=32, kv_heads=8, head_dim=128, n_req=1, ctx=32768,
                       hit=1.0, query=28, n_docs=1),
    "llama70b32k": dict(name="llama3-70b_1x32k", layers=80, kv_heads=8, head_dim=128, n_req=1, ctx=32768,
                        hit=1.0, query=28, n_docs=1),
}


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def cpu_model() -> str:
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return "unknown"


# ------------------------------------------------------------------------------------------------
# self-launch: `python bench.py --gpus N` without torchrun starts N ranks itself
# ------------------------------------------------------------------------------------------------
def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(args) -> int:
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", str(Path(__file__).resolve())] + sys.argv[1:]
    env = dict(os.environ)
    if args.one_device:
        env["TSB_BENCH_ONE_DEVICE"] = "1"
    return subprocess.call(cmd, env=env)


# ------------------------------------------------------------------------------------------------
# clocks during the timed region
# ------------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap", "utilization.gpu"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            threading.Thread(target=self._read, daemon=True).start()
            t0 = time.time()  # a timed region shorter than the sampling period still gets the first sample
            while not self.lines and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = [r for r in self.lines if len(r) == len(self.FIELDS)]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------------------------------------
# pools
# ------------------------------------------------------------------------------------------------
def make_pool(shape_full, n_slots, world, rank, dist, seed, kind, device):
    """The L2 pool this rank reads.  kind:
      numa   (default) pinned memory bound to the GPU's NUMA node (tsb_pool_create_numa).  With
             N > 1 ranks each rank holds only its KV heads (chunks [L][2][C][H/N][D]), so the box
             holds one pool's worth of host memory and every link reads its own socket's DIMMs.
      shared one /dev/shm segment of full chunks page-locked by every rank (strided head reads)
      hostalloc  cudaHostAlloc portable|mapped (round-1 default; N = 1 only)
    Returns (pool, description, shape the rank ingests with, seed of the pool contents)."""
    from paper_2603_21257_b200 import ingest

    node = ingest.device_numa_node(device)
    if kind == "shared" and world > 1:
        from paper_2603_21257_b200.multirank import SharedSegment

        nbytes = n_slots * shape_full.chunk_bytes
        if not torch_tensor_flag(SharedSegment.fits(nbytes), dist):
            raise SystemExit("--pool shared: /dev/shm cannot hold the pool")
        seg = SharedSegment(f"tsb_pool_{os.environ.get('MASTER_PORT', '0')}_{nbytes}", nbytes, rank, dist.barrier)
        pool = ingest.ChunkPool.register(shape_full, seg.address(), n_slots, keepalive=seg)
        if rank == 0:
            pool.fill_synthetic(seed)
        dist.barrier()
        seg.unlink()  # every rank has mapped and registered it: nothing outlives the run
        return pool, "shared /dev/shm segment of full chunks, cudaHostRegister'ed by every rank", \
            shape_full.with_rank(world, rank), seed
    def create_numa(shape):
        # mbind can be refused (a container's seccomp policy): place the pages by first touch then
        try:
            return ingest.ChunkPool.create_numa(shape, n_slots, node)
        except Exception as e:  # noqa: BLE001
            if node < 0:
                raise
            print(f"[bench] NUMA binding to node {node} refused ({e}); default placement", file=sys.stderr)
            return ingest.ChunkPool.create_numa(shape, n_slots, -1)

    if world > 1:
        local = ingest.KVShape(shape_full.layers, shape_full.kv_heads // world, shape_full.head_dim,
                               shape_full.dtype_bytes, shape_full.chunk_tokens, shape_full.page_tokens)
        pool = create_numa(local)
        pool.fill_synthetic(seed + rank)
        return pool, f"rank-local pinned pool of this rank's KV heads on NUMA node {pool.numa_node} " \
                     f"(GPU's node {node}; tsb_pool_create_numa)", local, seed + rank
    if kind == "hostalloc":
        pool = ingest.ChunkPool(shape_full, n_slots)
        desc = "cudaHostAlloc portable|mapped"
    else:
        pool = create_numa(shape_full)
        desc = f"pinned pool on NUMA node {pool.numa_node} (GPU's node {node}; tsb_pool_create_numa)"
    pool.fill_synthetic(seed)
    return pool, desc, shape_full, seed


def coll_device(dist) -> str:
    """Device of the tensors the timing/agreement collectives use: CUDA under NCCL, host under gloo."""
    return "cpu" if dist is not None and dist.get_backend() == "gloo" else "cuda"


def torch_tensor_flag(flag: bool, dist) -> bool:
    """All ranks agree on a boolean (logical AND over ranks)."""
    import torch

    t = torch.tensor([1 if flag else 0], device=coll_device(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def measure_ce_peak(torch, reps=5):
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    best = 1e9
    for i in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        d.copy_(h, non_blocking=True)
        b.record()
        b.synchronize()
        if i:
            best = min(best, a.elapsed_time(b) * 1e-3)
    del h, d
    return n / best / 1e9


def measure_k2(torch, l1, shape, n_items=128, reps=20):
    """K2 (k_ingest_ldg over the CE staging ring) timed alone with CUDA events on its stream, on
    the launch shape the CE path issues: n_items chunks x as many consecutive layers as one
    512 MiB staging half holds, each item's slice of this rank's heads packed.  Algorithmic bytes
    = read + write of that payload."""
    from paper_2603_21257_b200 import _capi, ingest
    from paper_2603_21257_b200.tiersim import check

    cb = shape.page_bytes * shape.pages_per_chunk
    rid = 1 << 40
    for c in range(n_items):
        g, row = l1.request(rid, c, cb)
        assert g
    l1.sync_block_table()
    local_layer = 2 * shape.chunk_tokens * shape.heads_local * shape.head_dim * shape.dtype_bytes
    n_layers = max(1, min(shape.layers - 1, (512 << 20) // (n_items * local_layer)))
    staging = torch.empty(n_items * n_layers * local_layer, dtype=torch.uint8, device="cuda")
    items = ingest.items_numpy(np.arange(n_items), [row] * n_items, np.arange(n_items))
    dev_items = torch.from_numpy(items.view(np.uint8).copy()).cuda()
    s = torch.cuda.current_stream()
    launch = lambda: check(_capi.lib.tsb_scatter_device_packed(l1.handle, staging.data_ptr(), dev_items.data_ptr(),
                                                                n_items, 1, 1 + n_layers, s.cuda_stream))
    for _ in range(3):
        launch()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        launch()
    b.record(s)
    b.synchronize()
    avg_s = a.elapsed_time(b) * 1e-3 / reps
    l1.release_request(rid)
    del staging
    return 2 * n_items * n_layers * local_layer, avg_s


def measure_k8(torch, l1, shape, n_items, reps=10):
    """K8 (tsb_l1_copy_chunks, HBM -> HBM chunk replication) timed alone with CUDA events: n_items
    chunks of one row copied into another row, all layers; algorithmic bytes = read + write."""
    from paper_2603_21257_b200 import _capi
    from paper_2603_21257_b200.tiersim import check

    cb = shape.page_bytes * shape.pages_per_chunk
    ra = rb = -1
    for c in range(n_items):
        g, ra = l1.request((1 << 40) + 2, c, cb)
        assert g
    for c in range(n_items):
        g, rb = l1.request((1 << 40) + 3, c, cb)
        assert g
    l1.sync_block_table()
    items = (_capi.PageCopy * n_items)(*[_capi.PageCopy(ra, c, rb, c) for c in range(n_items)])
    s = torch.cuda.current_stream()
    launch = lambda: check(_capi.lib.tsb_l1_copy_chunks(l1.handle, items, n_items, 0, shape.layers, s.cuda_stream))
    for _ in range(3):
        launch()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        launch()
    b.record(s)
    b.synchronize()
    l1.release_request((1 << 40) + 3)
    l1.release_request((1 << 40) + 2)
    return 2 * n_items * shape.local_chunk_bytes, a.elapsed_time(b) * 1e-3 / reps


def measure_k1_hbm(torch, l1, pool, shape, n_items, reps=10):
    """K1 (k_ingest_ldg, HBM grid) reading the HBM-resident pool, timed alone with CUDA events:
    layers [1, L) of a request's n_items chunks; algorithmic bytes = read + write of the payload."""
    from paper_2603_21257_b200 import ingest

    cb = shape.page_bytes * shape.pages_per_chunk
    rid = (1 << 40) + 1
    for c in range(n_items):
        g, row = l1.request(rid, c, cb)
        assert g
    l1.sync_block_table()
    items = ingest.items_numpy(np.arange(n_items) % pool.n_slots, [row] * n_items, np.arange(n_items))
    dev_items = torch.from_numpy(items.view(np.uint8).copy()).cuda()
    s = torch.cuda.current_stream()
    lo = 1 if shape.layers > 1 else 0
    launch = lambda: ingest.ingest_device(l1, pool, dev_items, n_items, lo, shape.layers, mode=ingest.ZEROCOPY,
                                          stream=s)
    for _ in range(3):
        launch()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        launch()
    b.record(s)
    b.synchronize()
    avg_s = a.elapsed_time(b) * 1e-3 / reps
    l1.release_request(rid)
    layer_bytes = 2 * shape.chunk_tokens * shape.heads_local * shape.head_dim * shape.dtype_bytes
    return 2 * n_items * (shape.layers - lo) * layer_bytes, avg_s


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def scaled_traffic(summary_name, alg_bytes):
    """dram read+write bytes of one launch from a committed `ncu --set full` summary, scaled from
    the profiled launch's algorithmic bytes to this launch's (null when not captured)."""
    p = ROOT / "profiles" / summary_name
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    dram, alg = d.get("dram_bytes_per_launch"), d.get("algorithmic_bytes_per_launch")
    return dram * alg_bytes / alg if dram and alg else None


# ------------------------------------------------------------------------------------------------
# CPU arm (oracle port, test infrastructure): numpy + oracle/ only, never the product package
# ------------------------------------------------------------------------------------------------
class _Shape:
    def __init__(self, layers, kv_heads, head_dim, dtype_bytes=2, chunk_tokens=256, page_tokens=16, tp_size=1,
                 tp_rank=0):
        self.__dict__.update(locals())
        del self.__dict__["self"]
        self.heads_local = kv_heads // tp_size
        self.chunk_bytes = layers * 2 * chunk_tokens * kv_heads * head_dim * dtype_bytes
        self.local_chunk_bytes = self.chunk_bytes // tp_size
        self.pages_per_chunk = chunk_tokens // page_tokens


def reference_sample(spec, per_request: int):
    """The configs batch in the oracle's FIFO pick order, cut to its first `per_request` chunks
    per request: (shape, items, block_table, num_pages, distinct pool slots used)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle as po

    shape = _Shape(spec["layers"], spec["kv_heads"], spec["head_dim"])
    n = spec["n_req"]
    nb = int(np.floor(spec["ctx"] * spec["hit"] / 256.0))  # cached_token_count (types.cpp:73-79)
    ids = np.arange(1, n + 1, dtype=np.int64)
    arrival = np.arange(n) * 1e-3
    order = po.sort_order(arrival, arrival, ids)  # FIFO: primary = arrival (scheduler.cpp:47-49)
    k = min(per_request, nb)
    # slot s of document d holds chunk s; request r reads document r % n_docs
    slots_used = sorted({(r % spec["n_docs"]) * k + c for r in range(n) for c in range(k)})
    remap = {s: i for i, s in enumerate(slots_used)}
    items = np.zeros(n * k, dtype=[("src_slot", np.int64), ("bt_row", np.int32), ("chunk_index", np.int32)])
    for j, r in enumerate(order):
        for c in range(k):
            items[j * k + c] = (remap[(int(r) % spec["n_docs"]) * k + c], j, c)
    num_pages = n * k * shape.pages_per_chunk
    bt = np.random.default_rng(5).permutation(num_pages).astype(np.int32).reshape(n, k * shape.pages_per_chunk)
    return shape, items, bt, num_pages, len(slots_used)


def cpu_scatter(shape, pool_view, items, bt, num_pages, threads, arena):
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle as po

    t0 = time.perf_counter()
    po.scatter_ref(shape, pool_view, items, bt, num_pages, threads=threads, arena=arena)
    return time.perf_counter() - t0


def run_reference(args):
    """The reference's CPU implementation of the path on the host cores: the reference moves no
    bytes (proj/ is a simulator), so this is the oracle port scatter_ref over the same batch in
    the same pick order, all host threads, one bounded sample per step."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle as po

    spec = SPECS[args.workload]
    threads = os.cpu_count() or 1
    shape, items, bt, num_pages, n_slots = reference_sample(spec, args.cpu_chunks_per_request)
    pool_view = po.synth_fill(7, 0, n_slots * shape.chunk_bytes // 8, threads).view(np.uint8)
    arena = np.empty(shape.layers * 2 * num_pages * 16 * shape.heads_local * shape.head_dim * 2, np.uint8)
    nbytes = len(items) * shape.local_chunk_bytes
    times = []
    for i in range(args.warmup + args.steps):
        secs = cpu_scatter(shape, pool_view, items, bt, num_pages, threads, arena)
        if i >= args.warmup:
            times.append(secs)
    tot = sum(times)
    value = args.steps * nbytes / tot / 1e9
    desc = (f"{spec['name']} batch in FIFO pick order, first {len(items) // spec['n_req']} chunks of each of the "
            f"{spec['n_req']} requests per step ({len(items)} chunks, {nbytes / 1e9:.2f} GB; pool {n_slots} slots), "
            f"oracle scatter_ref into paged L1 through a permuted block_table, {threads} threads")
    cpu = {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc, "cpu_model": cpu_model()}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": spec["name"], "sample": desc, "same_batch_as_ours": True},
            "impl": "reference", "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------------
def timed_steps(torch, run, steps, dist, capi):
    """W warm-up steps are run by the caller; this times exactly `steps` calls of `run()`,
    bracketed by a barrier + synchronize on both sides.  Returns (device s, wall s, last result,
    kernel launches, clocks)."""
    dev = torch.cuda.current_device()
    s = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    walls, results = [], None
    # The sampler starts (and delivers its first sample) before the barrier, so every rank leaves
    # the barrier straight into its timed region: no start skew between ranks.
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        launches0 = capi.lib.tsb_kernel_launch_count()
        ev0.record(s)
        for _ in range(steps):
            t0 = time.perf_counter()
            results = run()
            walls.append(time.perf_counter() - t0)
        ev1.record(s)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = capi.lib.tsb_kernel_launch_count() - launches0
    return ev0.elapsed_time(ev1) * 1e-3, sum(walls), results, launches, clk.summary()


def stage_pass(torch, wl, shape, pool, pool_seed, steps, warmup, l1_gib, layout=0, mode=None, dist=None,
               policy=None, hbm_tier_pool=None, tier_chunks=0, reuse_l1=False):
    """Warm-up (the first pass checks every page against the synthetic generator) + `steps` timed
    stage passes over the workload's batch on `pool`.  Returns a dict of the measurements and the
    L1 (the caller frees it)."""
    from paper_2603_21257_b200 import _capi, ingest
    from paper_2603_21257_b200.stage import LoadStage
    from paper_2603_21257_b200.tiersim import PolicyKind

    mode = ingest.AUTO if mode is None else mode
    policy = PolicyKind.Fifo if policy is None else policy
    free, _ = torch.cuda.mem_get_info()
    page = shape.page_bytes
    need_pages = wl.chunks * shape.pages_per_chunk
    num_pages = int(min((min(free - (10 << 30), l1_gib << 30)) // page, need_pages))
    max_chunks = max(len(s) for s in wl.slots)
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=wl.queue.n + 1, max_chunks=max(max_chunks, 128),
                             layout=layout)
    stage = LoadStage(l1, pool)
    slots = wl.slots
    if hbm_tier_pool is not None and tier_chunks:
        stage.set_hbm_tier(hbm_tier_pool)
        slots = [[~s if k < tier_chunks else s for k, s in enumerate(sl)] for sl in wl.slots]
    run = lambda verify=0: stage.run(wl.queue, slots, wl.config, policy=policy, mode=mode, verify_seed=verify,
                                     reuse_l1=reuse_l1)
    for i in range(warmup):
        r = run(pool_seed if i == 0 else 0)
        if i == 0 and r.stats["verify_mismatches"]:
            raise SystemExit(f"ingest parity failure ({wl.name}): {r.stats['verify_mismatches']} mismatching words")
    dev_s, wall_s, res, launches, clk = timed_steps(torch, run, steps, dist, _capi)
    req = res.requests
    order = np.argsort(req["pick_position"])
    out = dict(dev_s=dev_s, wall_s=wall_s, bytes=float(res.stats["bytes"]), launches=int(launches), clocks=clk,
               stats={k: res.stats[k] for k in ("ingest_calls", "deferred_chunks", "releases", "kernel_launches",
                                                "reused_chunks")},
               num_pages=num_pages, page=page, max_chunks=max_chunks,
               ttft={"first_layer_ms_p50": float(np.median(req["first_layer_ms"])),
                     "resident_ms_p50": float(np.median(req["resident_ms"])),
                     "resident_ms_max": float(req["resident_ms"].max()),
                     "first_layer_ms_first_request": float(req["first_layer_ms"][order[0]]),
                     "resident_ms_first_request": float(req["resident_ms"][order[0]]),
                     "reference_model_ms_per_request": float(
                         len(wl.slots[0]) * (10e-6 + shape.local_chunk_bytes / 64e9) * 1e3)})
    stage.close()
    return out, l1


def side_workloads(torch, args, ce_peak, hbm_peak, seed, device):
    """configs[0], configs[2] (rank 0 of tp 1/2/4/8 on this GPU) and configs[4] as sub-lines."""
    from paper_2603_21257_b200 import ingest
    from paper_2603_21257_b200.workloads import WORKLOADS

    out = {}
    steps = max(3, min(args.steps, 10))
    for key, tps in (("llama8b32k", (1,)), ("llama70b32k", (1, 2, 4, 8))):
        wl = WORKLOADS[key]()
        pool, desc, _, pseed = make_pool(wl.shape, wl.pool_slots, 1, 0, None, seed, "numa", device)
        for tp in tps:
            # rank 0 of a tp-way split.  `value`: the rank-local pool `bench.py --gpus tp` gives each
            # rank (its heads only, contiguous); `shared_pool`: the same rank reading its head slice
            # out of full chunks (strided copies; the /dev/shm shared-segment deployment)
            runs = {}
            for which in (("local", "shared") if tp > 1 else ("local",)):
                if which == "local" and tp > 1:
                    p_use, _, shape, p_seed = make_pool(wl.shape, wl.pool_slots, tp, 0, None, seed, "numa", device)
                else:
                    p_use, shape, p_seed = pool, wl.shape.with_rank(tp, 0), pseed
                m, l1 = stage_pass(torch, wl, shape, p_use, p_seed, steps, 3, 100)
                runs[which] = m
                del l1
                if p_use is not pool:
                    p_use.close()
                torch.cuda.empty_cache()
            m = runs["local"]
            link = m["bytes"] * steps / m["dev_s"] / 1e9
            out[f"{wl.name}" + (f"_tp{tp}_rank0" if tp > 1 else "")] = {
                "config": "configs[0]" if key == "llama8b32k" else f"configs[2] tp{tp} (rank 0 on this GPU)",
                "value": link, "e2e": m["bytes"] * steps / m["wall_s"] / 1e9, "unit": UNIT,
                "host_link_frac": link / ce_peak, "bytes_per_step": int(m["bytes"]),
                "ms_per_step": m["dev_s"] / steps * 1e3, "ttft_load_ms": m["ttft"], "steps": steps,
                "gpu_launches": m["launches"],
                "pool": "rank-local (this rank's heads)" if tp > 1 else "full chunks"}
            if "shared" in runs:
                ms = runs["shared"]
                sl = ms["bytes"] * steps / ms["dev_s"] / 1e9
                out[f"{wl.name}_tp{tp}_rank0"]["shared_pool"] = {
                    "value": sl, "e2e": ms["bytes"] * steps / ms["wall_s"] / 1e9, "host_link_frac": sl / ce_peak,
                    "pool": "full chunks, strided head-slice copies"}
        pool.close()
    out["mixed_trace"] = mixed_workload(torch, ce_peak, device)
    try:
        out["layer_pipelining"] = pipelining_workload(torch, ce_peak, device)
    except Exception as e:  # noqa: BLE001  the third-party consumer (FlashInfer JIT) failed: no
        # fallback, the sub-line reports why and the contract line stands
        out["layer_pipelining"] = {"skipped": f"real consumer unavailable: {type(e).__name__}: {e}"}
    out["queue100k"] = queue_workload(torch, hbm_peak)
    return out


def pipelining_workload(torch, ce_peak, device, n=12, ctx=32768, hit=0.97):
    """SURVEY f1 on the driver's line: 12 requests of 32K tokens at 0.97 hit (Llama-3.1-8B KV, one
    request's ingest ~ its prefill), the real consumer (PagedPrefill: FlashInfer paged prefill over
    the ingested pages + Llama-8B bf16 GEMMs) as the stage's prefill hook; ingest alone, prefill
    after residency, and layer-pipelined on per-layer fences.  Every page verified in the warm-up."""
    from paper_2603_21257_b200 import ingest
    from paper_2603_21257_b200 import tiersim as t
    from paper_2603_21257_b200.consumer import PagedPrefill
    from paper_2603_21257_b200.stage import LoadStage

    shape = ingest.LLAMA31_8B
    nb = int(np.floor(ctx * hit / shape.chunk_tokens))
    q = t.QueueArrays(n, id=np.arange(1, n + 1), arrival=np.arange(n) * 1e-6, context_tokens=np.full(n, ctx),
                      query_tokens=np.full(n, 28), cache_hit_ratio=np.full(n, hit), flags=np.zeros(n, np.uint8))
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(32, 8, 128, 2))
    pool = ingest.ChunkPool.create_numa(shape, nb, ingest.device_numa_node(device))
    pool.fill_synthetic(9)
    slots = [list(range(nb))] * n  # LooGLE-like: the requests share one document
    l1 = ingest.PagedKVCache(shape, n * nb * shape.pages_per_chunk + 64, max_rows=n + 1, max_chunks=nb)
    stage = LoadStage(l1, pool)
    first = stage.run(q, slots, cfg, verify_seed=9)
    consumer = PagedPrefill(l1, q, cfg)
    stage.set_prefill_hook(consumer)
    stage.run(q, slots, cfg, prefill=True, layer_events=True)  # FlashInfer / cuBLAS warm-up
    runs = {}
    for name, kw in (("ingest_only", {}), ("serial_prefill", dict(prefill=True)),
                     ("layer_pipelined_prefill", dict(prefill=True, layer_events=True))):
        stage.set_prefill_hook(consumer if kw else None)
        r = stage.run(q, slots, cfg, **kw).requests
        runs[name] = {"ttft_ms_mean": float((r["done_ms"] - r["arrival_ms"]).mean()),
                      "resident_ms_mean": float(r["resident_ms"].mean()), "batch_ms": float(r["done_ms"].max()),
                      "ingest_GBps": n * nb * shape.local_chunk_bytes / (r["resident_ms"].max() * 1e-3) / 1e9}
    out = {"config": "SURVEY f1 (configs[3] shape, balanced batch)", "requests": n, "context_tokens": ctx,
           "hit_ratio": hit, "verify_mismatches": int(first.stats["verify_mismatches"]), "runs": runs,
           "consumer": "PagedPrefill: FlashInfer paged prefill over l1.layer(l) + Llama-3.1-8B bf16 GEMMs",
           "ttft_reduction": 1.0 - runs["layer_pipelined_prefill"]["ttft_ms_mean"] / runs["serial_prefill"]["ttft_ms_mean"],
           "host_link_frac": runs["ingest_only"]["ingest_GBps"] / ce_peak}
    stage.close()
    del consumer, l1
    pool.close()
    torch.cuda.empty_cache()
    return out


def mixed_workload(torch, ce_peak, device, n=48, seed=0):
    """configs[3]: 2K-128K prefixes (lognormal mean 24K, cv 1.0, the product's generate_workload),
    hits {0.25, 0.5, 0.75, 0.9, 1.0}, Llama-3.1-8B KV; ingest alone, then with K6 prefill at a
    B200-like 4 us/token, serial (prefill after residency) and layer-pipelined (per-layer fences);
    TTFT of each, and the reference DES's TTFT for the same batch at the measured link rate."""
    from paper_2603_21257_b200 import ingest
    from paper_2603_21257_b200 import tiersim as t
    from paper_2603_21257_b200.stage import LoadStage

    spec = t.WorkloadSpec(t.DatasetProfile("mixed", n, 24000.0, 1.0, 28.0, 0.0), qps=1e6, count=n, seed=seed,
                          hit_ratio_source=t.HitRatioSource.uniform_choice([0.25, 0.5, 0.75, 0.9, 1.0]))
    q = t.generate_queue(spec)
    q.context_tokens[:] = np.clip(q.context_tokens, 2048, 131072)
    shape = ingest.LLAMA31_8B
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(32, 8, 128, 2), compute_per_token=4e-6)
    plans = [int(np.floor(q.context_tokens[i] * q.cache_hit_ratio[i] / 256)) for i in range(n)]
    n_slots = max(plans) + 64
    pool = ingest.ChunkPool.create_numa(shape, n_slots, ingest.device_numa_node(device))
    pool.fill_synthetic(5)
    rng = np.random.default_rng(3)
    slots = [list(range(s0, s0 + nb)) for nb in plans for s0 in [int(rng.integers(0, n_slots - nb + 1))]]
    num_pages = (80 << 30) // shape.page_bytes
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=n + 1, max_chunks=max(plans) + 1)
    stage = LoadStage(l1, pool)
    first = stage.run(q, slots, cfg, verify_seed=5)
    out = {"config": "configs[3]", "requests": n, "chunks": int(sum(plans)),
           "bytes": int(sum(plans) * shape.local_chunk_bytes), "verify_mismatches": int(first.stats["verify_mismatches"])}
    runs = {}
    for name, kw in (("ingest_only", {}), ("serial_prefill", dict(prefill=True)),
                     ("overlapped_prefill", dict(prefill=True, layer_events=True))):
        r = stage.run(q, slots, cfg, **kw)
        req = r.requests
        runs[name] = {"batch_ms": float(req["done_ms"].max()),
                      "ingest_GBps": r.stats["bytes"] / (req["resident_ms"].max() * 1e-3) / 1e9,
                      "ttft_ms_mean": float(req["done_ms"].mean()), "ttft_ms_p50": float(np.median(req["done_ms"]))}
        runs[name]["_req"] = req
    out["runs"] = {k: {kk: vv for kk, vv in v.items() if kk != "_req"} for k, v in runs.items()}
    out["host_link_frac"] = runs["ingest_only"]["ingest_GBps"] / ce_peak
    out["overlap_gain"] = runs["serial_prefill"]["batch_ms"] / runs["overlapped_prefill"]["batch_ms"]
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle as po

    if po.ref() is not None:  # the reference DES of the same batch, at the measured link rate
        rate = runs["ingest_only"]["ingest_GBps"] * 1e9
        sim = t.ClusterConfig(bytes_per_token=cfg.bytes_per_token, network_bandwidth=1e18, pcie_bandwidth=rate,
                              transfer_base_latency=0.0, l1_capacity=num_pages * shape.page_bytes, l2_capacity=10**15,
                              compute_per_token=cfg.compute_per_token, compute_base=cfg.compute_base)
        m = t.cost_models_from_config(sim)
        ttft = np.zeros(n)
        mean = C.c_double()
        st = po.ref().ref_run_simulation(n, C.byref(po.queue_struct(q)), C.byref(po.cluster_struct(sim)), 0,
                                         (C.c_double * 4)(m.load.slope, m.load.intercept, m.comp.slope,
                                                          m.comp.intercept), 0, ttft.ctypes.data, C.byref(mean))
        if st == 0:
            real = runs["serial_prefill"]["_req"]["done_ms"] * 1e-3
            err = np.abs(real - ttft) / ttft
            out["sim_vs_real"] = {"sim_mean_ttft_ms": mean.value * 1e3, "real_mean_ttft_ms": float(real.mean() * 1e3),
                                  "mean_abs_rel_err": float(err.mean()), "max_abs_rel_err": float(err.max()),
                                  "cpu_baseline_kind": "reference"}
    stage.close()
    del l1
    pool.close()
    torch.cuda.empty_cache()
    return out


def queue_workload(torch, hbm_peak, n=100_000):
    """configs[4]: generate_workload(loogle, 100K, seed 0) + assign_slos {2,4,8} (the product's own
    generator), GPU score + order for 5 policies, K3 prefix hashing of every context, K7 index."""
    from paper_2603_21257_b200 import hasher
    from paper_2603_21257_b200 import tiersim as t
    from paper_2603_21257_b200.scorer import BatchScorer, DeviceQueue

    spec = t.WorkloadSpec(t.builtin_profile("loogle"), qps=1.0, count=n, seed=0)
    t0 = time.perf_counter()
    q = t.generate_queue(spec)
    cfg = t.ClusterConfig(l1_capacity=10**13, l2_capacity=10**13)
    t.assign_slos_queue(q, cfg, [2.0, 4.0, 8.0], 0)
    gen_s = time.perf_counter() - t0
    m = t.cost_models_from_config(cfg)
    sc = BatchScorer(torch.cuda.current_device())
    dq = DeviceQueue(q, torch.cuda.current_device())
    out = sc.score_device(dq, t.PolicyKind.Lstf, m, cfg)

    def timed(fn, reps=20, warm=3):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) * 1e-3 / reps

    gpu = {t.policy_name(p): timed(lambda: sc.score_device(dq, p, m, cfg, out=out, check_errors=False)) * 1e6
           for p in t.PolicyKind}
    sc.score(q, t.PolicyKind.Lstf, m, cfg)
    t0 = time.perf_counter()
    for _ in range(5):
        order = sc.score(q, t.PolicyKind.Lstf, m, cfg)[3]
    api_us = (time.perf_counter() - t0) / 5 * 1e6
    res = {"config": "configs[4]", "requests": n, "queue_generation_s": gen_s,
           "gpu_score_order_us": gpu, "host_api_score_order_us": api_us}
    # K3 over every context of the queue; token ids generated on the device (doc-id prefixes shared).
    # Requests sit at 16-byte-aligned starts (gaps of <= 3 tokens): the layout K3 reads with whole
    # 16-byte vectors; the chunk counts come from the true lengths, so the hashes are the same.
    offs = hasher.aligned_offsets(q.context_tokens)
    dev = torch.device("cuda", torch.cuda.current_device())
    d_offs = torch.from_numpy(offs).to(dev)
    doc = torch.from_numpy(np.random.default_rng(1).integers(0, 1000, n)).to(dev)
    sh = torch.from_numpy(q.context_tokens // 2).to(dev)
    tok = torch.empty(int(offs[-1]), dtype=torch.int32, device=dev)
    hasher.gen_tokens_device(0, d_offs, doc, sh, tok)
    coff = torch.from_numpy(hasher.chunk_offsets_of_lengths(q.context_tokens)).to(dev)
    hout = torch.empty(int(coff[-1]), dtype=torch.int64, device=dev)
    secs = timed(lambda: hasher.hash_prefix_chunks_device(d_offs, tok, coff, hout), reps=10)
    p1 = timed(lambda: hasher.chunk_digests_device(d_offs, tok, coff, hout), reps=10)
    hasher.hash_prefix_chunks_device(d_offs, tok, coff, hout)
    ntok = int(q.context_tokens.sum())
    nbytes = ntok * 4 + hout.numel() * 8
    read_ceiling = 7410.0  # read-only HBM ceiling measured on this pool (profiles/r01_hbm_read_probe.jsonl)
    res["hash"] = {"tokens": ntok, "chunks": int(coff[-1]), "ms": secs * 1e3, "GBps": nbytes / secs / 1e9,
                   "read_ceiling_GBps": read_ceiling, "read_ceiling_frac": nbytes / secs / 1e9 / read_ceiling,
                   "phase1_ms": p1 * 1e3, "phase1_read_ceiling_frac": nbytes / p1 / 1e9 / read_ceiling,
                   "hbm_copy_peak_frac": nbytes / secs / 1e9 / hbm_peak, "algorithmic_bytes": int(nbytes),
                   "layout": "16-byte-aligned request starts"}
    # CPU leg for the hash: the oracle restatement (hash_ref) over the first requests of the same
    # queue on all host threads and on one, checked equal to the GPU hashes of those requests
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle as po

    k = 4000
    lens = q.context_tokens[:k]
    tok_h = tok[: int(offs[k])].cpu().numpy()
    packed = np.concatenate([tok_h[offs[r]: offs[r] + lens[r]] for r in range(k)])
    p_offs = np.zeros(k + 1, np.int64)
    np.cumsum(lens, out=p_offs[1:])
    threads = os.cpu_count() or 1
    cpu_hash = {}
    for th in (threads, 1):
        t0 = time.perf_counter()
        h_cpu = po.hash_prefix_chunks(p_offs, packed, threads=th)
        cpu_hash[th] = time.perf_counter() - t0
    sample_bytes = int(lens.sum()) * 4 + h_cpu.size * 8
    res["hash"]["cpu_baseline"] = {
        "kind": "port", "cores": threads, "cpu_model": cpu_model(),
        "GBps": sample_bytes / cpu_hash[threads] / 1e9, "GBps_1_thread": sample_bytes / cpu_hash[1] / 1e9,
        "sample": f"first {k} requests of the queue ({int(lens.sum())} tokens), oracle hash_ref",
        "equal_to_gpu": bool(np.array_equal(h_cpu, hout[: int(coff[k])].cpu().numpy().view(np.uint64)))}
    del tok_h, packed
    idx = hasher.PrefixIndex(capacity=1 << int(np.ceil(np.log2(2 * hout.numel()))))
    slots_t = torch.arange(hout.numel(), dtype=torch.int64, device=dev)
    ins_s = timed(lambda: idx.insert_device(hout, slots_t), reps=1, warm=0)
    m_out = torch.empty(n, dtype=torch.int64, device=dev)
    s_out = torch.empty_like(hout)
    look_s = timed(lambda: idx.lookup_device(coff, hout, s_out, m_out), reps=10)
    res["index"] = {"insert_ms": ins_s * 1e3, "lookup_ms": look_s * 1e3, "lookups_per_s": hout.numel() / look_s}
    # the reference's own scorer + sort on one core (oracle/_ref; the cpu_baseline leg), when built
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle as po

    mm = [m.load.slope, m.load.intercept, m.comp.slope, m.comp.intercept]
    if po.ref() is not None:
        t0 = time.perf_counter()
        ref_order = po.ref_sort_order(q, int(t.PolicyKind.Lstf), mm, cfg)
        res["cpu_baseline"] = {"kind": "reference", "cores": 1, "cpu_model": cpu_model(),
                               "score_plus_sort_us": (time.perf_counter() - t0) * 1e6,
                               "sample": "the full 100K queue, LSTF: estimate_service_cost + priority_key + "
                                         "std::sort(PriorityKey::operator<) of the compiled reference"}
        res["order_equal_reference"] = bool(np.array_equal(order, ref_order))
    del tok, hout, s_out, idx
    torch.cuda.empty_cache()
    return res


def run_ours(args):
    import torch

    rank, world, local = env_rank()
    dist = None
    if world > 1:
        import torch.distributed as tdist

        # TSB_BENCH_ONE_DEVICE=1 (a validation mode, not a measurement): every rank on cuda:0 over
        # gloo, to exercise the multi-rank path (pools, head shards, reductions) on one GPU.
        one_dev = os.environ.get("TSB_BENCH_ONE_DEVICE") == "1"
        local = 0 if one_dev else local
        torch.cuda.set_device(local)
        if one_dev:
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    from paper_2603_21257_b200 import ingest
    from paper_2603_21257_b200.multirank import reduce_timing
    from paper_2603_21257_b200.stage import LoadStage
    from paper_2603_21257_b200.tiersim import PolicyKind
    from paper_2603_21257_b200.workloads import WORKLOADS

    wl = WORKLOADS[args.workload]()
    wl.for_rank(world, rank)  # validates the head split
    seed = 20261017
    ce_peak = measure_ce_peak(torch)
    pool, pool_kind, shape, pool_seed = make_pool(wl.shape, wl.pool_slots, world, rank, dist, seed, args.pool, dev)
    if args.emulate_tp > 1:  # one GPU standing in for rank 0 of a TP-sharded box (configs[2])
        if world > 1:
            raise SystemExit("--emulate-tp is for single-GPU runs")
        shape = wl.shape.with_rank(args.emulate_tp, 0)
    hbm_peak, hbm_src = measured_peaks()

    # ---- value + e2e: the north-star hop, pinned host pool -> L1 pages ---------------------------
    m, l1 = stage_pass(torch, wl, shape, pool, pool_seed, args.steps, args.warmup, args.l1_gib,
                       layout=ingest.LAYOUTS[args.layout], mode=ingest.MODES[args.mode], dist=dist)
    local_bytes = m["bytes"]
    dev_s, wall_s, total_bytes = reduce_timing(dist, m["dev_s"], m["wall_s"], local_bytes, device=coll_device(dist))
    value = args.steps * total_bytes / dev_s / 1e9
    e2e = args.steps * total_bytes / wall_s / 1e9
    link_rate = args.steps * local_bytes / m["dev_s"] / 1e9  # this rank's link

    # the hand-written SM ingest kernels on the same stage, first 2 requests: K1 (16-byte zero-copy
    # loads) and K1b (cp.async.bulk); AUTO picks CE+K2 for host pools (SM reads cap at ~92.5%)
    modes = {}
    if not args.no_alt_modes:
        stage_host = LoadStage(l1, pool)
        s = torch.cuda.current_stream()
        sub = type(wl.queue)(2, **{k: getattr(wl.queue, k)[:2] for k, _ in type(wl.queue).FIELDS})
        for name in (("bulk", "zerocopy", "ce") if args.layout == "flashinfer_hnd" or shape.tp_size > 1
                     else ("bulk", "zerocopy", "ce", "ce_direct")):
            stage_host.run(sub, wl.slots[:2], wl.config, mode=ingest.MODES[name])  # warm
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            r = stage_host.run(sub, wl.slots[:2], wl.config, mode=ingest.MODES[name])
            b.record(s)
            b.synchronize()
            gbs = r.stats["bytes"] / (a.elapsed_time(b) * 1e-3) / 1e9
            modes[name] = {"GBps": gbs, "host_link_frac": gbs / ce_peak}
        stage_host.close()
        del stage_host
        if dist:
            dist.barrier()

    # K2 (the CE path's paged scatter, HBM-bound), measured live on the stage's group size
    layer_bytes = 2 * shape.chunk_tokens * shape.heads_local * shape.head_dim * shape.dtype_bytes
    k2_items = min((512 << 20) // layer_bytes, m["max_chunks"])
    k2_alg, k2_s = measure_k2(torch, l1, shape, n_items=k2_items)
    k2_roof = {"bound": "hbm", "kernel": "k_ingest_ldg (K2 paged scatter from the CE staging ring, one staging group)",
               "achieved": k2_alg / k2_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
               "frac": k2_alg / k2_s / 1e9 / hbm_peak, "traffic": scaled_traffic("k2_ncu_summary.json", k2_alg),
               "peak_source": hbm_src, "algorithmic_bytes_per_launch": int(k2_alg), "launch_us": k2_s * 1e6,
               "share_of_step": None}
    roofline = {"bound": "host_link",
                "kernel": "L2->L1 hop: copy engines (cudaMemcpy2DAsync per run of consecutive pool slots into the HBM staging ring) + K2 paged "
                          "scatter; achieved = this GPU's payload bytes over the link / CUDA-event time of the passes",
                "achieved": link_rate, "peak": ce_peak, "unit": "GB/s", "frac": link_rate / ce_peak,
                "traffic": None, "peak_source": "live pinned 1 GiB cudaMemcpy H2D, best of 5, this box",
                "theory_gen5_x16_gbs": GEN5_X16_GBS, "frac_of_theory": link_rate / GEN5_X16_GBS,
                "algorithmic_bytes": "payload read from the host pool once (local chunk bytes x chunks)",
                "k2_hbm_frac": k2_roof["frac"]}

    # ---- l1_reuse: the same step, chunks already resident in a live request's pages replicated
    # HBM -> HBM (K8) instead of crossing the link again (not the headline) ----------------------
    l1_reuse = None
    if not args.no_l1_reuse:
        del l1
        torch.cuda.empty_cache()
        rm, l1 = stage_pass(torch, wl, shape, pool, pool_seed, args.steps, min(args.warmup, 3), args.l1_gib,
                            layout=ingest.LAYOUTS[args.layout], mode=ingest.MODES[args.mode], dist=dist, reuse_l1=True)
        r_s, r_wall, r_bytes = reduce_timing(dist, rm["dev_s"], rm["wall_s"], rm["bytes"], device=coll_device(dist))
        reused = rm["stats"]["reused_chunks"]
        k8_items = max(1, min(rm["max_chunks"], rm["num_pages"] // (2 * shape.pages_per_chunk)))
        k8_alg, k8_s = measure_k8(torch, l1, shape, k8_items)
        hbm_peak8, _ = measured_peaks()
        l1_reuse = {"value": args.steps * r_bytes / r_s / 1e9, "e2e": args.steps * r_bytes / r_wall / 1e9, "unit": UNIT,
                    "ms_per_step": r_s / args.steps * 1e3, "reused_chunks_per_step": reused,
                    "link_bytes_per_step": int(rm["bytes"] - reused * shape.local_chunk_bytes),
                    "link_GBps": (rm["bytes"] - reused * shape.local_chunk_bytes) * args.steps / rm["dev_s"] / 1e9,
                    "delivered_bytes_per_step": int(rm["bytes"]), "ttft_load_ms": rm["ttft"],
                    "gpu_launches": rm["launches"],
                    "roofline_k8": {"bound": "hbm", "kernel": "k_page_copy (K8: chunk replication inside L1)",
                                    "achieved": k8_alg / k8_s / 1e9, "peak": hbm_peak8, "unit": "GB/s",
                                    "frac": k8_alg / k8_s / 1e9 / hbm_peak8, "algorithmic_bytes_per_launch": int(k8_alg),
                                    "launch_us": k8_s * 1e6, "chunks_per_launch": k8_items},
                    "source": "stage option reuse_l1: a chunk whose L2 slot is resident in a live request's pages is "
                              "copied HBM -> HBM by K8 (tsb_l1_copy_chunks); every page verified in the warm-up"}

    # ---- hbm_tier: the same step with the pool in HBM (peer-HBM tier kernel path, K1) -----------
    hbm_tier = None
    if not args.no_hbm_tier:
        free, _ = torch.cuda.mem_get_info()
        l1_bytes = m["num_pages"] * m["page"]
        if wl.pool_slots * pool.shape.chunk_bytes + (24 << 30) < free + l1_bytes:
            del l1
            torch.cuda.empty_cache()
            dpool = ingest.ChunkPool.create_device(pool.shape, wl.pool_slots, device=dev)
            dpool.fill_synthetic(pool_seed)
            hm, l1 = stage_pass(torch, wl, shape, dpool, pool_seed, args.steps, min(args.warmup, 3), args.l1_gib,
                                layout=ingest.LAYOUTS[args.layout], dist=dist)
            h_s, _, h_bytes = reduce_timing(dist, hm["dev_s"], hm["wall_s"], hm["bytes"], device=coll_device(dist))
            k1_alg, k1_s = measure_k1_hbm(torch, l1, dpool, shape, hm["max_chunks"])
            hbm_tier = {"value": args.steps * h_bytes / h_s / 1e9, "unit": UNIT,
                        "ms_per_step": h_s / args.steps * 1e3, "gpu_launches": hm["launches"], "clocks": hm["clocks"],
                        "source": "the same L2 pool slots held in this GPU's HBM (tsb_pool_create_device), CUDA events",
                        "roofline": {"bound": "hbm", "kernel": "k_ingest_ldg (K1 over the HBM-resident pool)",
                                     "achieved": k1_alg / k1_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                                     "frac": k1_alg / k1_s / 1e9 / hbm_peak,
                                     "traffic": scaled_traffic("k1hbm_ncu_summary.json", k1_alg),
                                     "algorithmic_bytes_per_launch": int(k1_alg), "launch_us": k1_s * 1e6}}
            dpool.close()
    del l1
    torch.cuda.empty_cache()

    bt_bytes = wl.queue.n * (max(m["max_chunks"], 128) * shape.pages_per_chunk) * 4
    cfg = {"workload": wl.name, "description": wl.description,
           "parallelism": (f"kv-head shards tp{world}" if world > 1 else
                           f"single GPU as rank 0 of a tp{args.emulate_tp} head split" if args.emulate_tp > 1
                           else "single GPU"),
           "ingest_mode": args.mode, "policy": "fifo", "l1_layout": args.layout, "l1_pages": m["num_pages"],
           "l1_page_bytes": m["page"], "l1_gib": round(m["num_pages"] * m["page"] / 2**30, 1),
           "bytes_per_step": int(total_bytes), "pool": pool_kind,
           "l2_flush": "inputs larger than L2 (each step streams the whole batch: 100s of GB)",
           "value_source": "L2 pool in pinned host memory; CUDA events on the stage stream around the K passes",
           "stage": m["stats"]}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dev_s / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic", "config": cfg,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(local_bytes + bt_bytes + wl.queue.n * 66),
                "d2h_bytes_per_step": int(wl.queue.n * (8 + 16)),
                "source": "host wall time of the public-API calls (tsb_stage_run) over the same K passes: queue "
                          "and block-table uploads, ingest, results read back; the KV payload is the H2D traffic"},
        "gpu_launches": m["launches"], "roofline": roofline, "roofline_k2": k2_roof,
        "host_link": {"achieved": link_rate, "peak": ce_peak, "frac": link_rate / ce_peak, "unit": UNIT},
        "ttft_load_ms": m["ttft"], "clocks": m["clocks"], "ingest_modes_2req": modes, "hbm_tier": hbm_tier,
        "l1_reuse": l1_reuse,
    }
    if world == 1 and not args.no_side and args.workload == "qwen16x128k" and args.emulate_tp == 1:
        pool.close()
        line["workloads"] = side_workloads(torch, args, ce_peak, hbm_peak, seed, dev)
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        spec = SPECS[args.workload]
        shp, items, bt, num_pages, n_slots = reference_sample(spec, args.cpu_chunks_per_request)
        sys.path.insert(0, str(ROOT / "oracle"))
        import pyoracle as po

        view = po.synth_fill(7, 0, n_slots * shp.chunk_bytes // 8, threads).view(np.uint8)
        arena = np.empty(shp.layers * 2 * num_pages * 16 * shp.heads_local * shp.head_dim * 2, np.uint8)
        cpu_scatter(shp, view, items, bt, num_pages, threads, arena)  # first touch
        times = []
        while len(times) < 2 or sum(times) < 10.0:
            times.append(cpu_scatter(shp, view, items, bt, num_pages, threads, arena))
        nbytes = len(items) * shp.local_chunk_bytes
        q1 = max(1, len(items) // 8)  # one thread over an eighth of the sample (same pick order)
        one = cpu_scatter(shp, view, items[:q1], bt, num_pages, 1, arena)
        line["cpu_baseline"] = {"value": nbytes * len(times) / sum(times) / 1e9, "unit": UNIT, "cores": threads,
                                "kind": "port", "cpu_model": cpu_model(),
                                "value_1_thread": q1 * shp.local_chunk_bytes / one / 1e9,
                                "sample": f"{len(items)} chunks ({nbytes / 1e9:.2f} GB) of the {spec['name']} batch "
                                          f"in FIFO pick order, oracle scatter_ref, {threads} threads, "
                                          f"{len(times)} passes over >= 10 s of CPU work (mean)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="qwen16x128k", choices=sorted(SPECS))
    ap.add_argument("--mode", default="auto", choices=["auto", "ce", "bulk", "zerocopy"])
    ap.add_argument("--pool", default="numa", choices=["numa", "shared", "hostalloc"])
    ap.add_argument("--l1-gib", type=int, default=100)
    ap.add_argument("--layout", default="flash_attn", choices=["flash_attn", "flashinfer_nhd", "flashinfer_hnd"],
                    help="the consumer's L1 page layout")
    ap.add_argument("--emulate-tp", type=int, default=1, help="one GPU ingests rank 0's head slice of a tpN split")
    ap.add_argument("--one-device", action="store_true",
                    help="validation: with --gpus N > 1, every rank on cuda:0 over gloo (not a measurement)")
    ap.add_argument("--no-hbm-tier", action="store_true", help="skip the HBM-resident-pool arm")
    ap.add_argument("--no-l1-reuse", action="store_true", help="skip the reuse_l1 arm")
    ap.add_argument("--no-side", action="store_true", help="skip the configs[0]/[2]/[4] sub-lines")
    ap.add_argument("--cpu-chunks-per-request", type=int, default=32)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-alt-modes", action="store_true", help="skip the K1/K1b/CE side measurements")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "ours" and not args.one_device:
            import torch

            if torch.cuda.device_count() < args.gpus:
                raise SystemExit(f"--gpus {args.gpus}: only {torch.cuda.device_count()} GPUs visible "
                                 f"(--one-device runs every rank on cuda:0 as a validation)")
        sys.exit(launch_ranks(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
