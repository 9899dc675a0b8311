#!/usr/bin/env python3
"""Contract benchmark: KV ingest GB/s (L2 pinned host chunk pool -> L1 paged HBM) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload ...]

A step is one pass of the load stage over the batch: GPU scoring + pick order, TierLedger-
semantics page grants with FIFO deferral, block-table upload, ingest of every planned chunk, and
page release (tsb_stage_run, the public C-ABI call).  Default workload = BASELINE.json configs[1]
(Qwen2.5-32B KV, 16 x 128K @ 0.9 hit).  With N GPUs the KV heads are sharded TP-style: every rank
ingests its head slice of the same batch from the pool (strong scaling, no data-path collective).

  value : inputs resident in HBM -- the same L2 pool (slots, bytes) held in device memory; payload
          bytes of all ranks / max over ranks of the CUDA-event time of the K timed stage passes
  e2e   : the L2 pool in pinned host memory, so every payload byte crosses the host link inside
          the timed region; the same bytes / max over ranks of the host wall time of the K
          public-API calls (the headline against the reference arm)
  roofline     : the value arm's dominant kernel (K1 over the HBM pool, HBM-bound), live CUDA events
  roofline_k2  : the e2e arm's kernel (K2 paged scatter from the CE staging ring)
  host_link    : the e2e arm's device-timed GB/s per GPU vs the live copy-engine H2D peak
  cpu_baseline : the oracle's scatter_ref (port) on the host cores, bounded sample (rank 0, N=1)
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
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


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


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
# shared pool across per-GPU processes
# ------------------------------------------------------------------------------------------------
def make_pool(shape_full, n_slots, world, rank, dist, seed):
    """One pinned L2 pool per box: a /dev/shm segment page-locked by every rank when it fits;
    otherwise each rank pins a shard-local pool holding only its KV heads (chunks laid out
    [L][2][C][H/world][D]), so host memory stays at one pool's worth across the box.
    Returns (pool, description, shape the rank ingests with)."""
    from paper_2603_21257_b200 import ingest
    from paper_2603_21257_b200.multirank import SharedSegment

    nbytes = n_slots * shape_full.chunk_bytes
    if world > 1:
        shared = torch_tensor_flag(SharedSegment.fits(nbytes), dist)
        if shared:
            seg = SharedSegment(f"tsb_pool_{os.environ.get('MASTER_PORT', '0')}_{nbytes}", nbytes, rank, dist.barrier)
            pool = ingest.ChunkPool.register(shape_full, seg.address(), n_slots, keepalive=seg)
            if rank == 0:
                pool.fill_synthetic(seed)
            dist.barrier()
            seg.unlink()  # every rank has mapped and registered it: nothing outlives the run
            return pool, "shared /dev/shm segment, cudaHostRegister'ed by every rank", shape_full.with_rank(world, rank)
        local = ingest.KVShape(shape_full.layers, shape_full.kv_heads // world, shape_full.head_dim,
                               shape_full.dtype_bytes, shape_full.chunk_tokens, shape_full.page_tokens)
        pool = ingest.ChunkPool(local, n_slots)
        pool.fill_synthetic(seed + rank)
        return pool, "shard-local pinned pool per rank (/dev/shm too small for one shared pool)", local
    pool = ingest.ChunkPool(shape_full, n_slots)
    pool.fill_synthetic(seed)
    return pool, "cudaHostAlloc portable|mapped", shape_full


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
# CPU baseline (oracle port, test infrastructure) -- rank 0, N = 1 only
# ------------------------------------------------------------------------------------------------
def cpu_scatter_baseline(shape, sample_chunks, seed, threads, reps=2, pool_view=None, min_seconds=0.0):
    """scatter_ref over `sample_chunks` chunks, `reps` timed passes (more until min_seconds of
    CPU work): returns (GB/s over all timed passes, bytes per pass, mean seconds per pass)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle as po

    cb = shape.chunk_bytes
    if pool_view is None:
        pool_view = po.synth_fill(seed, 0, sample_chunks * cb // 8, threads).view(np.uint8)
    num_pages = sample_chunks * shape.pages_per_chunk
    rng = np.random.default_rng(seed)
    bt = rng.permutation(num_pages).astype(np.int32).reshape(1, -1)
    items = np.zeros(sample_chunks, dtype=[("src_slot", np.int64), ("bt_row", np.int32), ("chunk_index", np.int32)])
    items["src_slot"] = np.arange(sample_chunks)
    items["chunk_index"] = np.arange(sample_chunks)
    arena = np.empty(shape.layers * 2 * num_pages * shape.page_tokens * shape.heads_local * shape.head_dim
                     * shape.dtype_bytes, np.uint8)
    po.scatter_ref(shape, pool_view, items, bt, num_pages, threads=threads, arena=arena)  # first touch
    times = []
    while len(times) < reps or sum(times) < min_seconds:
        t0 = time.perf_counter()
        po.scatter_ref(shape, pool_view, items, bt, num_pages, threads=threads, arena=arena)
        times.append(time.perf_counter() - t0)
    nbytes = sample_chunks * shape.local_chunk_bytes
    mean = sum(times) / len(times)
    return nbytes / mean / 1e9, nbytes, mean


# ------------------------------------------------------------------------------------------------
def run_reference(args):
    """The reference CPU implementation of the path on the host cores: the reference moves no
    bytes (proj/ is a simulator), so this is the oracle port scatter_ref over the same chunk
    layouts, all host threads, one bounded sample per step."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from paper_2603_21257_b200.workloads import WORKLOADS

    wl = WORKLOADS[args.workload]()
    shape = wl.shape
    threads = os.cpu_count() or 1
    sample = args.cpu_sample_chunks
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle as po

    pool_view = po.synth_fill(7, 0, sample * shape.chunk_bytes // 8, threads).view(np.uint8)
    times = []
    for i in range(args.warmup + args.steps):
        gbs, nbytes, secs = cpu_scatter_baseline(shape, sample, 7, threads, reps=1, pool_view=pool_view)
        if i >= args.warmup:
            times.append(secs)
    tot = sum(times)
    value = args.steps * nbytes / tot / 1e9
    desc = f"{sample} chunks ({nbytes / 1e9:.2f} GB) of request 1 of {wl.name}, scatter_ref, {threads} threads"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": wl.name, "sample": desc},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


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


def measure_k1_hbm(torch, l1, pool, shape, n_items, reps=10):
    """K1 (k_ingest_ldg, K2 grid) reading the HBM-resident pool, timed alone with CUDA events:
    the stage's dominant launch -- layers [1, L) of a request's n_items chunks (layer 0 goes
    first, alone, to fence the first layer); algorithmic bytes = read + write of the payload."""
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


def run_ours(args):
    import torch

    rank, world, local = env_rank()
    dist = None
    if world > 1:
        import torch.distributed as tdist

        # TSB_BENCH_ONE_DEVICE=1 (a validation mode, not a measurement): every rank on cuda:0 over
        # gloo, to exercise the multi-rank path (shared pool, head shards, reductions) on one GPU.
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
    from paper_2603_21257_b200 import _capi, ingest
    from paper_2603_21257_b200.multirank import reduce_timing
    from paper_2603_21257_b200.stage import LoadStage
    from paper_2603_21257_b200.tiersim import PolicyKind
    from paper_2603_21257_b200.workloads import WORKLOADS

    wl = WORKLOADS[args.workload]()
    wl.for_rank(world, rank)  # validates the head split
    seed = 20261017
    ce_peak = measure_ce_peak(torch)
    pool, pool_kind, shape = make_pool(wl.shape, wl.pool_slots, world, rank, dist, seed)
    pool_seed = seed + rank if shape.tp_size == 1 and world > 1 else seed
    pool_shape = pool.shape
    if args.emulate_tp > 1:  # one GPU standing in for rank 0 of a TP-sharded box (configs[2])
        if world > 1:
            raise SystemExit("--emulate-tp is for single-GPU runs")
        shape = wl.shape.with_rank(args.emulate_tp, 0)

    # The same L2 pool resident in this GPU's HBM (same slot layout and contents): the `value` arm.
    dpool = None
    if not args.no_hbm_arm:
        free, _ = torch.cuda.mem_get_info()
        if wl.pool_slots * pool_shape.chunk_bytes + (40 << 30) < free:
            dpool = ingest.ChunkPool.create_device(pool_shape, wl.pool_slots, device=dev)
            dpool.fill_synthetic(pool_seed)

    # L1 arena: most of the remaining HBM, fewer pages than the batch needs so FIFO deferral is
    # exercised.  Both arms share it.
    free, total = torch.cuda.mem_get_info()
    page = shape.page_bytes
    need_pages = wl.chunks * shape.pages_per_chunk
    arena_bytes = min(free - (10 << 30), args.l1_gib << 30)
    num_pages = min(arena_bytes // page, need_pages)
    max_chunks = max(len(s) for s in wl.slots)
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=wl.queue.n + 1, max_chunks=max(max_chunks, 128),
                             layout=ingest.LAYOUTS[args.layout])
    mode = ingest.MODES[args.mode]
    stage_host = LoadStage(l1, pool)
    host_slots, tier_chunks = wl.slots, 0
    if args.hbm_tier_chunks > 0:
        # The first K chunks of every request are already resident in an HBM tier (the value arm's
        # device pool, which holds every slot): they bypass the host link (tsb_ingest_tiered).
        if dpool is None:
            raise SystemExit("--hbm-tier-chunks needs the HBM arm's device pool")
        host_slots = [[~s if k < args.hbm_tier_chunks else s for k, s in enumerate(sl)] for sl in wl.slots]
        tier_chunks = sum(min(args.hbm_tier_chunks, len(sl)) for sl in wl.slots)
    run_host = lambda verify=0: stage_host.run(wl.queue, host_slots, wl.config, policy=PolicyKind.Fifo, mode=mode,
                                               verify_seed=verify)

    # ---- value: L2 pool resident in HBM, CUDA events around K stage passes ----------------------
    hbm = None
    if dpool is not None:
        stage_dev = LoadStage(l1, dpool)
        run_dev = lambda verify=0: stage_dev.run(wl.queue, wl.slots, wl.config, policy=PolicyKind.Fifo,
                                                 verify_seed=verify)
        for i in range(args.warmup):
            r = run_dev(pool_seed if i == 0 else 0)
            if i == 0 and r.stats["verify_mismatches"]:
                raise SystemExit(f"ingest parity failure (HBM pool): {r.stats['verify_mismatches']} words")
        d_s, d_wall, d_res, d_launch, d_clk = timed_steps(torch, run_dev, args.steps, dist, _capi)
        d_s, d_wall, d_bytes = reduce_timing(dist, d_s, d_wall, float(d_res.stats["bytes"]),
                                             device=coll_device(dist))
        k1_items = max_chunks
        k1_alg, k1_s = measure_k1_hbm(torch, l1, dpool, shape, k1_items)
        hbm = dict(dev_s=d_s, bytes=d_bytes, launches=d_launch, clocks=d_clk, stats=d_res.stats,
                   k1_alg=k1_alg, k1_s=k1_s, k1_items=k1_items)
        stage_dev.close()
        if args.hbm_tier_chunks > 0:
            stage_host.set_hbm_tier(dpool)
        else:
            dpool.close()
        torch.cuda.synchronize()

    # ---- e2e: pinned host pool, every byte crosses the host link inside the timed region -------
    for i in range(args.warmup):
        r = run_host(pool_seed if i == 0 else 0)  # the first one checks every page
        if i == 0 and r.stats["verify_mismatches"]:
            raise SystemExit(f"ingest parity failure: {r.stats['verify_mismatches']} mismatching words")
    h_s, wall_s, results, h_launch, h_clk = timed_steps(torch, run_host, args.steps, dist, _capi)
    local_bytes = results.stats["bytes"]
    link_bytes = local_bytes - tier_chunks * shape.local_chunk_bytes  # what crossed the host link
    h_s, wall_s, total_bytes = reduce_timing(dist, h_s, wall_s, float(local_bytes), device=coll_device(dist))
    host_dev_rate = args.steps * total_bytes / h_s / 1e9
    e2e = args.steps * total_bytes / wall_s / 1e9

    # The hand-written SM ingest kernels on the same stage, first 2 requests of the batch: K1
    # (16-byte zero-copy loads) and K1b (cp.async.bulk / TMA engine).  AUTO picks CE+K2 for
    # full-head chunks because SM-initiated host reads cap at ~92.6% of the copy-engine rate.
    s = torch.cuda.current_stream()
    modes = {}
    if not args.no_alt_modes:
        sub = type(wl.queue)(2, **{k: getattr(wl.queue, k)[:2] for k, _ in type(wl.queue).FIELDS})
        for name in (("zerocopy", "ce") if args.layout == "flashinfer_hnd" else ("bulk", "zerocopy", "ce")):
            stage_host.run(sub, wl.slots[:2], wl.config, mode=ingest.MODES[name])  # warm
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            r = stage_host.run(sub, wl.slots[:2], wl.config, mode=ingest.MODES[name])
            b.record(s)
            b.synchronize()
            modes[name] = {"GBps": r.stats["bytes"] / (a.elapsed_time(b) * 1e-3) / 1e9,
                           "host_link_frac": r.stats["bytes"] / (a.elapsed_time(b) * 1e-3) / 1e9 / ce_peak}
        if dist:
            dist.barrier()

    # K2 (the CE path's paged scatter, HBM-bound), measured live on the stage's group size
    layer_bytes = 2 * shape.chunk_tokens * shape.heads_local * shape.head_dim * shape.dtype_bytes
    k2_items = min((512 << 20) // layer_bytes, max_chunks)  # items of one request in a staging half
    k2_alg, k2_s = measure_k2(torch, l1, shape, n_items=k2_items)
    hbm_peak, hbm_src = measured_peaks()
    k2_traffic = scaled_traffic("k2_ncu_summary.json", k2_alg)
    k2_roof = {"bound": "hbm", "kernel": "k_ingest_ldg (K2 paged scatter from the CE staging ring, one staging group)",
               "achieved": k2_alg / k2_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
               "frac": k2_alg / k2_s / 1e9 / hbm_peak, "traffic": k2_traffic, "peak_source": hbm_src,
               "algorithmic_bytes_per_launch": int(k2_alg), "launch_us": k2_s * 1e6}
    req = results.requests
    order = np.argsort(req["pick_position"])
    ttft = {"first_layer_ms_p50": float(np.median(req["first_layer_ms"])),
            "resident_ms_p50": float(np.median(req["resident_ms"])),
            "resident_ms_max": float(req["resident_ms"].max()),
            "resident_ms_first_request": float(req["resident_ms"][order[0]]),
            "reference_model_ms_per_request": float(len(wl.slots[0]) * (10e-6 + shape.local_chunk_bytes / 64e9) * 1e3)}
    bt_bytes = wl.queue.n * l1.stride * 4
    link_rate = host_dev_rate / world * link_bytes / local_bytes
    host_link = {"achieved": link_rate, "peak": ce_peak, "unit": "GB/s",
                 "frac": link_rate / ce_peak, "ms_per_step": h_s / args.steps * 1e3,
                 "peak_source": "live pinned 1 GiB cudaMemcpy H2D, best of 5, this box",
                 "kernel_launches": int(h_launch)}
    e2e_obj = {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(link_bytes + bt_bytes + wl.queue.n * 66),
               "d2h_bytes_per_step": int(wl.queue.n * (8 + 16)),
               "source": "L2 pool in pinned host memory (" + pool_kind + "); host wall time of the public-API "
                         "calls (tsb_stage_run); the KV payload is the H2D traffic"}
    cfg = {"workload": wl.name, "description": wl.description,
           "hbm_tier": ({"chunks_per_step": tier_chunks, "bytes_per_step": int(tier_chunks * shape.local_chunk_bytes),
                         "note": "first K chunks of every request resident in an HBM tier (tsb_ingest_tiered); "
                                 "e2e counts all delivered bytes, h2d only the host-link part"}
                        if tier_chunks else None),
           "parallelism": (f"kv-head shards tp{world}" if world > 1 else
                           f"single GPU as rank 0 of a tp{args.emulate_tp} head split" if args.emulate_tp > 1
                           else "single GPU"),
           "ingest_mode": args.mode, "policy": "fifo", "l1_layout": args.layout, "l1_pages": int(num_pages),
           "l1_page_bytes": int(page), "l1_gib": round(num_pages * page / 2**30, 1),
           "bytes_per_step": int(total_bytes), "pool": pool_kind,
           "l2_flush": "inputs larger than L2 (each step streams the whole batch: 100s of GB)"}
    if hbm is not None:
        value = args.steps * hbm["bytes"] / hbm["dev_s"] / 1e9
        ms_per_step = hbm["dev_s"] / args.steps * 1e3
        launches = hbm["launches"]
        clocks = hbm["clocks"]
        k1_traffic = scaled_traffic("k1hbm_ncu_summary.json", hbm["k1_alg"])
        roofline = {"bound": "hbm", "kernel": "k_ingest_ldg (K1 over the HBM-resident pool, 4736 CTAs, 4 loads in flight per lane)",
                    "achieved": hbm["k1_alg"] / hbm["k1_s"] / 1e9, "peak": hbm_peak, "unit": "GB/s",
                    "frac": hbm["k1_alg"] / hbm["k1_s"] / 1e9 / hbm_peak, "traffic": k1_traffic,
                    "peak_source": hbm_src, "algorithmic_bytes_per_launch": int(hbm["k1_alg"]),
                    "launch_us": hbm["k1_s"] * 1e6, "items_per_launch": hbm["k1_items"],
                    "algorithmic_bytes": "read + write of the payload (2 x chunks x layers [1, L) x layer slice)"}
        cfg["value_source"] = ("L2 pool resident in HBM (tsb_pool_create_device, same slots and bytes); "
                               "CUDA events on the stage stream around the K passes")
        cfg["hbm_arm_stage"] = {k: hbm["stats"][k] for k in ("ingest_calls", "deferred_chunks", "releases",
                                                             "kernel_launches")}
    else:  # HBM cannot hold pool + L1: value falls back to the host-pool device time
        value, ms_per_step, launches, clocks, roofline = host_dev_rate, h_s / args.steps * 1e3, h_launch, h_clk, k2_roof
        cfg["value_source"] = "L2 pool in pinned host memory (HBM too small for the pool); CUDA events"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic", "config": cfg,
        "e2e": e2e_obj, "gpu_launches": int(launches), "roofline": roofline,
        "roofline_k2": k2_roof, "host_link": host_link, "ttft_load_ms": ttft,
        "stage": {k: results.stats[k] for k in ("ingest_calls", "deferred_chunks", "releases", "kernel_launches")},
        "clocks": clocks, "clocks_e2e": h_clk,
        "ingest_modes_2req": modes,
    }
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sample = args.cpu_sample_chunks
        view = pool.slot_view(0, sample)
        gbs, nbytes, secs = cpu_scatter_baseline(wl.shape, sample, seed, threads, pool_view=view, min_seconds=10.0)
        passes = max(2, int(round(10.0 / secs)))
        line["cpu_baseline"] = {"value": gbs, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"{sample} chunks ({nbytes / 1e9:.2f} GB) of {wl.name} from the pinned "
                                          f"pool, oracle scatter_ref, {threads} threads, ~{passes} passes over "
                                          f">= 10 s of CPU work (mean)"}
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
    ap.add_argument("--workload", default="qwen16x128k")
    ap.add_argument("--mode", default="auto", choices=["auto", "ce", "bulk", "zerocopy"])
    ap.add_argument("--l1-gib", type=int, default=100)
    ap.add_argument("--layout", default="flash_attn", choices=["flash_attn", "flashinfer_nhd", "flashinfer_hnd"],
                    help="the consumer's L1 page layout")
    ap.add_argument("--hbm-tier-chunks", type=int, default=0,
                    help="e2e arm: the first K chunks of every request come from an HBM tier (not the headline)")
    ap.add_argument("--emulate-tp", type=int, default=1, help="one GPU ingests rank 0's head slice of a tpN split")
    ap.add_argument("--no-hbm-arm", action="store_true", help="skip the HBM-resident-pool arm (value)")
    ap.add_argument("--cpu-sample-chunks", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-alt-modes", action="store_true", help="skip the K1/K1b/CE side measurements")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        raise SystemExit(f"--gpus {args.gpus}: launch one process per GPU with "
                         f"`python -m torch.distributed.run --nproc-per-node {args.gpus} bench.py --gpus {args.gpus}`")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
