"""f2: close the loop from measured ingest (and real prefill) to the scheduler's cost model.

  1. calibration runs of the load stage over the stream's plans: per-request (cached tokens,
     ingest seconds) and, with the real PagedPrefill consumer and no layer pipelining,
     (compute tokens, prefill seconds) -> read_samples_csv-format CSVs -> fit_linear;
  2. the same request stream (the product's generate_workload, LooGLE profile, hits from
     {0.25, 0.5, 0.75, 1.0}; deadlines from assign_slos with the box's calibrated config) replayed
     in real time through tsb_stage_run_online under SJF-cost and LSTF, once with the reference's
     cost_models_from_config defaults and once with the fitted models;
  3. reports the fits, how far the static pick orders moved (Kendall distance), and mean TTFT /
     SLO attainment of each run.  Prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_21257_b200 import calibrate, ingest  # noqa: E402
from paper_2603_21257_b200 import tiersim as t  # noqa: E402
from paper_2603_21257_b200.scorer import BatchScorer  # noqa: E402
from paper_2603_21257_b200.stage import LoadStage  # noqa: E402


def kendall_distance(a, b):
    """Fraction of request pairs the two orders rank differently."""
    pos = np.empty(len(b), np.int64)
    pos[b] = np.arange(len(b))
    x = pos[a]
    n = len(x)
    inv = sum(int(np.sum(x[i + 1:] < x[i])) for i in range(n))
    return inv / max(1, n * (n - 1) // 2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=60)
    ap.add_argument("--qps", type=float, default=6.0)
    ap.add_argument("--consumer", choices=["real", "k6"], default="real")
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "calibration"))
    args = ap.parse_args()
    shape = ingest.LLAMA31_8B
    bpt = t.kv_bytes_per_token(32, 8, 128, 2)
    spec = t.WorkloadSpec(t.builtin_profile("loogle"), qps=args.qps, count=args.n, seed=1,
                          hit_ratio_source=t.HitRatioSource.uniform_choice([0.25, 0.5, 0.75, 1.0]))
    q = t.generate_queue(spec)
    q.context_tokens[:] = np.minimum(q.context_tokens, 131072)
    base = t.ClusterConfig(bytes_per_token=bpt, l1_capacity=10**13, l2_capacity=10**13)
    plans = [int(np.floor(q.context_tokens[i] * q.cache_hit_ratio[i] / 256)) for i in range(q.n)]
    n_slots = max(plans) + 32
    pool = ingest.ChunkPool(shape, n_slots)
    pool.fill_synthetic(3)
    rng = np.random.default_rng(2)
    slots = []
    for nb in plans:
        s0 = int(rng.integers(0, n_slots - nb + 1))
        slots.append(list(range(s0, s0 + nb)))
    num_pages = (60 << 30) // shape.page_bytes
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=q.n + 1, max_chunks=max(plans) + 1,
                             layout=ingest.LAYOUT_FLASHINFER_NHD)
    stage = LoadStage(l1, pool)
    consumer = None
    if args.consumer == "real":
        from paper_2603_21257_b200.consumer import PagedPrefill

        consumer = PagedPrefill(l1, q, base)
        stage.set_prefill_hook(consumer)

    # 1. calibration: the batch stage, prefill serial (starts at residency), twice (first warms JIT)
    stage.run(q, slots, base, prefill=True, verify_seed=3)
    cal_runs = [stage.run(q, slots, base, prefill=True) for _ in range(2)]
    cal = calibrate.calibrate(cal_runs, base, args.out, fit_compute=True)
    if consumer is not None:
        stage.set_prefill_hook(None)
    alone = stage.run(q, slots, base)  # ingest only: the link rate without prefill interference
    if consumer is not None:
        stage.set_prefill_hook(consumer)
    link = alone.stats["bytes"] / (alone.requests["resident_ms"].max() * 1e-3)
    box = t.ClusterConfig(bytes_per_token=bpt, l1_capacity=10**13, l2_capacity=10**13, network_bandwidth=1e15,
                          transfer_base_latency=0.0, pcie_bandwidth=bpt / cal.models.load.slope,
                          compute_per_token=cal.models.comp.slope, compute_base=cal.models.comp.intercept)
    t.assign_slos_queue(q, box, [2.0, 4.0, 8.0], 7)
    out = {"workload": f"{q.n} LooGLE-profile requests (product generate_workload, seed 1), {args.qps} QPS, hits "
                       "{0.25,0.5,0.75,1.0}, Llama-3.1-8B KV, deadlines assign_slos {2,4,8} x solo TTFT on this box",
           "consumer": args.consumer, "measured_link_GBps": link / 1e9,
           "fit": {"load": {"slope": cal.models.load.slope, "intercept": cal.models.load.intercept,
                            "slope_clamped": cal.load.slope_clamped, "intercept_clamped": cal.load.intercept_clamped,
                            "implied_GBps": bpt / cal.models.load.slope / 1e9},
                   "comp": {"slope": cal.models.comp.slope, "intercept": cal.models.comp.intercept}},
           "default": {"load": {"slope": cal.default.load.slope, "intercept": cal.default.load.intercept},
                       "comp": {"slope": cal.default.comp.slope, "intercept": cal.default.comp.intercept}},
           "samples_csv": [cal.load_csv, cal.comp_csv],
           "load_samples": {"used": sum(int(((r.requests["chunks"] > 0) & (r.requests["deferred_chunks"] == 0)).sum())
                                        for r in cal_runs),
                            "left_out_deferred": sum(int(((r.requests["chunks"] > 0) & (r.requests["deferred_chunks"] > 0)).sum())
                                                     for r in cal_runs)}}
    # 2. static orders under both models
    sc = BatchScorer(0)
    orders = {}
    for pol in (t.PolicyKind.SjfCost, t.PolicyKind.Lstf):
        od = sc.score(q, pol, cal.default, base)[3]
        oc = sc.score(q, pol, cal.models, base)[3]
        orders[t.policy_name(pol)] = {"kendall_distance": kendall_distance(od, oc),
                                      "first10_default": od[:10].tolist(), "first10_calibrated": oc[:10].tolist()}
    out["order_change"] = orders
    # 3. real-time replays
    runs = {}
    for pol in (t.PolicyKind.SjfCost, t.PolicyKind.Lstf, t.PolicyKind.Fifo):
        for name, models in (("default", cal.default), ("calibrated", cal.models)):
            if pol == t.PolicyKind.Fifo and name == "calibrated":
                continue
            r = stage.run_online(q, slots, base, models=models, policy=pol)
            ttft = (r.requests["done_ms"] - r.requests["arrival_ms"]) * 1e-3
            dl = q.deadline - q.arrival
            runs[f"{t.policy_name(pol)}/{name}"] = {"mean_ttft_s": float(ttft.mean()),
                                                   "p90_ttft_s": float(np.percentile(ttft, 90)),
                                                   "slo_attainment": float(np.mean(ttft <= dl))}
    out["online"] = runs
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
