"""configs[3]: mixed trace -- 2K-128K prefixes, varying hit ratios, ingest overlapped with
synthetic prefill (K6) -- plus the sim-vs-real comparison against the compiled reference DES.

Runs the load stage over a batch of LooGLE-like requests with the reference's compute model
(compute_base + compute_per_token * n) as K6 prefill, twice:
  * overlapped: per-layer fences, prefill of a request starts as its layers land;
  * serial: prefill waits for the request's last layer.
Then replays the same batch through tiersim_ref::run_simulation with pcie_bandwidth = the measured
ingest rate, no network stage and the same L1 capacity, and reports the per-request TTFT error.
Prints one JSON line.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
from paper_2603_21257_b200 import ingest  # noqa: E402
from paper_2603_21257_b200 import tiersim as t  # noqa: E402
from paper_2603_21257_b200.stage import LoadStage  # noqa: E402


def mixed_batch(n, seed, block=256):
    rng = np.random.default_rng(seed)
    sig = np.sqrt(np.log1p(1.0))  # cv 1.0 around a 24K mean, clamped to [2K, 128K]
    ctx = np.clip(np.round(np.exp(np.log(24000) - 0.5 * sig**2 + sig * rng.standard_normal(n))), 2048, 131072)
    ctx = ctx.astype(np.int64)
    hit = rng.choice([0.25, 0.5, 0.75, 0.9, 1.0], n)
    q = t.QueueArrays(n, id=np.arange(1, n + 1), arrival=np.zeros(n), context_tokens=ctx,
                      query_tokens=np.full(n, 28), cache_hit_ratio=hit, flags=np.zeros(n, np.uint8))
    q.arrival[:] = np.arange(n) * 1e-6  # all present; FIFO = index order
    return q


def stage_overlap(req, layer_events):
    """Device-clock spans from the stage's own CUDA events: ingest of request k is
    [ingest_begin, resident]; its prefill window is taken from the earliest it may start (its first
    layer when layer-pipelined, its residency when serial, and not before the previous prefill's
    end) to done.  Reports how long the link and those windows overlap, and how many requests were
    eligible to start prefill before they were fully resident.  These are inferred from the fences,
    not observed: whether prefill kernels actually ran early shows in the kineto timeline (--profile)
    and in the TTFT itself."""
    def union(iv):
        out = []
        for a, b in sorted(iv):
            if out and a <= out[-1][1]:
                out[-1] = (out[-1][0], max(out[-1][1], b))
            else:
                out.append((a, b))
        return out

    order = np.argsort(req["pick_position"], kind="stable")
    ingest = [(float(r["ingest_begin_ms"]), float(r["resident_ms"])) for r in req if r["chunks"] > 0]
    prefill, prev, early = [], 0.0, 0
    for k in order:
        r = req[k]
        ready = float(r["first_layer_ms"] if layer_events else r["resident_ms"])
        start = max(ready, prev)
        prefill.append((start, float(r["done_ms"])))
        early += int(start < float(r["resident_ms"]) - 1e-3)
        prev = float(r["done_ms"])
    ui, up = union(ingest), union(prefill)
    both = 0.0
    for a, b in ui:
        for c, d in up:
            both += max(0.0, min(b, d) - max(a, c))
    return {"link_busy_ms": sum(b - a for a, b in ui), "prefill_busy_ms": sum(b - a for a, b in up),
            "link_and_prefill_concurrent_ms": both, "prefills_eligible_before_own_residency": early,
            "source": "stage CUDA events (ingest_begin / first_layer / resident / done per request)"}


def timeline_summary(prof, path):
    """From a kineto (CUPTI) trace of one overlapped run: busy time of the ingest kernels (K2), of
    the host->device copies, of the prefill kernels, the ingest window [first K2 start, last K2 end],
    and how much prefill ran inside it."""
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    spans = {"ingest": [], "prefill": [], "memcpy": []}
    for e in ev:
        t0, t1 = e.time_range.start, e.time_range.end
        if "emcpy" in e.name:
            spans["memcpy"].append((t0, t1))
        elif "tsb::" in e.name:
            spans["ingest"].append((t0, t1))
        else:
            spans["prefill"].append((t0, t1))

    def union(iv):
        out = []
        for a, b in sorted(iv):
            if out and a <= out[-1][1]:
                out[-1] = (out[-1][0], max(out[-1][1], b))
            else:
                out.append((a, b))
        return out

    u = {k: union(v) for k, v in spans.items()}
    busy = {k: sum(b - a for a, b in v) / 1e3 for k, v in u.items()}
    w0 = min(a for a, _ in u["ingest"]) if u["ingest"] else 0
    w1 = max(b for _, b in u["ingest"]) if u["ingest"] else 0
    inside = sum(max(0, min(b, w1) - max(a, w0)) for a, b in u["prefill"]) / 1e3
    allt = [t for v in u.values() for iv in v for t in iv]
    res = {"source": "torch.profiler (kineto/CUPTI) CUDA activity of one overlapped run (nsys is not in the image)",
           "run_window_ms": (max(allt) - min(allt)) / 1e3 if allt else 0.0, "busy_ms": busy,
           "ingest_window_ms": (w1 - w0) / 1e3, "prefill_busy_inside_ingest_window_ms": inside,
           "prefill_share_of_ingest_window": inside / ((w1 - w0) / 1e3) if w1 > w0 else 0.0,
           "launches": {k: len(v) for k, v in spans.items()}}
    Path(path).write_text(json.dumps(res, indent=1))
    prof.export_chrome_trace(str(Path(path).with_suffix(".trace.json")))
    return res


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--compute-per-token", type=float, default=4e-5,
                    help="prefill seconds/token: 4e-5 = the reference calibration (types.hpp:91); "
                         "~4e-6 approximates an 8B prefill on B200")
    ap.add_argument("--consumer", choices=["k6", "real"], default="k6",
                    help="k6: the calibrated timer; real: PagedPrefill (FlashInfer paged attention over the "
                         "ingested pages + Llama-3.1-8B-sized bf16 GEMMs per layer) as the stage's prefill hook")
    ap.add_argument("--n", type=int, default=48)
    ap.add_argument("--uniform", default="", metavar="CTX:HIT",
                    help="instead of the mixed trace: n requests of CTX tokens at hit ratio HIT (e.g. 32768:0.9, "
                         "ingest and prefill of one request about equal on B200)")
    ap.add_argument("--mode", default="auto", choices=["auto", "ce", "ce_direct", "zerocopy", "bulk"],
                    help="the stage's ingest mode (AUTO: CE + K2 for the host pool)")
    ap.add_argument("--k2-ctas", type=int, default=0, help="K2 grid (0 = default 148 x 32)")
    ap.add_argument("--staging-mib", type=int, default=0, help="CE staging ring, both halves (0 = default 1024)")
    ap.add_argument("--profile", default="", help="write a kineto (CUPTI) timeline summary of the overlapped run here")
    args = ap.parse_args()
    shape = ingest.LLAMA31_8B
    n = args.n
    if args.k2_ctas:
        ingest.set_grid(scatter_ctas=args.k2_ctas)
    if args.staging_mib:
        ingest.set_ce(1, args.staging_mib << 20)
    if args.uniform:
        u_ctx, u_hit = args.uniform.split(":")
        q = mixed_batch(n, 0)
        q.context_tokens[:] = int(u_ctx)
        q.cache_hit_ratio[:] = float(u_hit)
    else:
        q = mixed_batch(n, 0)
    cfg = t.ClusterConfig(bytes_per_token=t.kv_bytes_per_token(32, 8, 128, 2),
                          compute_per_token=args.compute_per_token)
    plans = [int(np.floor(q.context_tokens[i] * q.cache_hit_ratio[i] / 256)) for i in range(n)]
    n_slots = max(plans) + 64
    pool = ingest.ChunkPool(shape, n_slots)
    pool.fill_synthetic(5)
    rng = np.random.default_rng(3)
    slots = []
    for nb in plans:  # each request's document starts somewhere in the pool (shared prefixes)
        s0 = int(rng.integers(0, n_slots - nb + 1))
        slots.append(list(range(s0, s0 + nb)))
    num_pages = 40 * 1024  # 80 GiB of L1 (80 GB GPU of the paper's setup, SPEC defaults)
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=n + 1, max_chunks=max(plans) + 1)
    stage = LoadStage(l1, pool)
    desc = (f"{n} requests of {args.uniform.split(':')[0]} tokens at hit {args.uniform.split(':')[1]}" if args.uniform
            else f"configs[3]: {n} requests, 2K-128K prefixes (lognormal mean 24K, cv 1.0), hit in {{0.25,0.5,0.75,0.9,1.0}}")
    out = {"workload": f"{desc}, Llama-3.1-8B KV, L1 {num_pages * shape.page_bytes / 2**30:.0f} GiB",
           "chunks": int(sum(plans)), "bytes": int(sum(plans) * shape.local_chunk_bytes), "ingest_mode": args.mode,
           "k2_ctas": args.k2_ctas or 148 * 32, "staging_mib": args.staging_mib or 1024,
           "max_connections": os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "default")}
    stage.run(q, slots, cfg, verify_seed=5)  # warm-up + full parity check
    consumer = None
    if args.consumer == "real":
        from paper_2603_21257_b200.consumer import PagedPrefill

        consumer = PagedPrefill(l1, q, cfg)
        stage.set_prefill_hook(consumer)
        stage.run(q, slots, cfg, prefill=True, layer_events=True)  # JIT + warm-up
        out["consumer"] = {"kind": "PagedPrefill: FlashInfer paged prefill attention over l1.layer(l) + "
                                   "Llama-3.1-8B-sized bf16 GEMMs (qkv, o, gate/up, down) per layer",
                           "tflop_per_batch": sum(consumer.flops_per_request(i) for i in range(n)) / 1e12}
    runs = {}
    for name, kw in (("ingest_only", dict(prefill=False)), ("serial_prefill", dict(prefill=True, layer_events=False)),
                     ("overlapped_prefill", dict(prefill=True, layer_events=True))):
        if consumer is not None and not kw.get("prefill"):
            stage.set_prefill_hook(None)
        if consumer is not None:
            consumer.host_s = consumer.host_max_s = consumer.plan_s = 0.0
        r = stage.run(q, slots, cfg, mode=ingest.MODES[args.mode], **kw)
        if consumer is not None:
            stage.set_prefill_hook(consumer)
        req = r.requests
        runs[name] = {"batch_ms": float(req["done_ms"].max()), "ingest_GBps": r.stats["bytes"] / (req["resident_ms"].max() * 1e-3) / 1e9,
                      "ttft_ms_mean": float(req["done_ms"].mean()), "ttft_ms_p50": float(np.median(req["done_ms"])),
                      "resident_ms_mean": float(req["resident_ms"].mean()), "deferred_chunks": r.stats["deferred_chunks"],
                      "wall_ms": r.stats["wall_ms"]}
        if consumer is not None and kw.get("prefill"):
            runs[name]["hook_host_ms"] = consumer.host_s * 1e3
            runs[name]["hook_host_max_ms"] = consumer.host_max_s * 1e3
            runs[name]["plan_host_ms"] = consumer.plan_s * 1e3
        runs[name]["_req"] = req
        if kw.get("prefill"):
            runs[name]["overlap"] = stage_overlap(req, kw.get("layer_events", False))
    out["runs"] = {k: {kk: vv for kk, vv in v.items() if kk != "_req"} for k, v in runs.items()}
    prefill_s = float(sum(cfg.compute_base + cfg.compute_per_token * (q.context_tokens[i] + 28 - plans[i] * 256)
                          for i in range(n)))
    out["prefill_total_ms"] = prefill_s * 1e3
    out["overlap_gain"] = runs["serial_prefill"]["batch_ms"] / runs["overlapped_prefill"]["batch_ms"]
    if consumer is not None:
        out["prefill_total_ms"] = None  # the real consumer's time is measured, not modelled
        out["real_ttft_mean_ms"] = {k: v["ttft_ms_mean"] for k, v in out["runs"].items() if k != "ingest_only"}
        out["ingest_GBps_with_prefill"] = runs["overlapped_prefill"]["ingest_GBps"]
        out["ingest_GBps_alone"] = runs["ingest_only"]["ingest_GBps"]
    if args.profile:
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            stage.run(q, slots, cfg, prefill=True, layer_events=True, mode=ingest.MODES[args.mode])
            torch.cuda.synchronize()
        out["timeline"] = timeline_summary(prof, args.profile)

    # sim-vs-real: the reference DES with the measured ingest rate, no network stage
    import pyoracle as po

    if po.ref() is not None:
        rate = runs["ingest_only"]["ingest_GBps"] * 1e9

        def des(compute_base, compute_per_token):
            sim_cfg = t.ClusterConfig(bytes_per_token=cfg.bytes_per_token, network_bandwidth=1e18, pcie_bandwidth=rate,
                                      transfer_base_latency=0.0, l1_capacity=num_pages * shape.page_bytes,
                                      l2_capacity=10**15, compute_base=compute_base, compute_per_token=compute_per_token)
            ttft = np.zeros(n)
            mean = C.c_double()
            models = t.cost_models_from_config(sim_cfg)
            st = po.ref().ref_run_simulation(n, C.byref(po.queue_struct(q)), C.byref(po.cluster_struct(sim_cfg)), 0,
                                             (C.c_double * 4)(models.load.slope, models.load.intercept,
                                                              models.comp.slope, models.comp.intercept),
                                             0, ttft.ctypes.data, C.byref(mean))
            if st != 0:
                return {"error": po.ref().ref_last_error().decode()}
            real = runs["serial_prefill"]["_req"]["done_ms"] * 1e-3
            err = np.abs(real - ttft) / ttft
            return {"sim_mean_ttft_ms": mean.value * 1e3, "real_mean_ttft_ms": float(real.mean() * 1e3),
                    "mean_abs_rel_err": float(err.mean()), "max_abs_rel_err": float(err.max()),
                    "compute_model": [compute_base, compute_per_token]}

        out["sim_vs_real"] = {"mode": "serial prefill vs DES (coupled stages per request are decoupled in both)",
                              **des(cfg.compute_base, cfg.compute_per_token)}
        if consumer is not None:
            # the real consumer's own cost: fit (compute tokens, prefill seconds) of the serial run
            from paper_2603_21257_b200 import calibrate

            samples = calibrate.compute_samples(runs["serial_prefill"]["_req"])
            if len({x.tokens for x in samples}) > 1:  # a uniform batch has one token count: no fit
                fit = t.fit_linear((x.tokens, x.seconds) for x in samples)
                out["sim_vs_real_calibrated"] = {"mode": "DES with T_comp fitted to this run's prefills (fit_linear)",
                                                 **des(fit.model.intercept, fit.model.slope)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
