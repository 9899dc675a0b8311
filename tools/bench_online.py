"""CALVO's scheduling experiment on real B200 ingest: a Poisson stream of LooGLE-like requests is
replayed in real time through tsb_stage_run_online under each policy (FIFO, SJF-PT, SJF-cost,
EDF, LSTF), and the same stream is run through the reference DES (tiersim_ref::run_simulation)
calibrated to the measured ingest rate.  Reports mean TTFT and SLO attainment, real vs simulated.

Stage mapping for the DES: our single transfer stage (pinned host pool -> paged HBM) plays the
DES's first stage, so network_bandwidth = measured ingest rate and the DES's PCIe hop is made
instantaneous; L1 capacity = our arena; compute = the K6 synthetic prefill's model.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
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


def loogle_stream(n, qps, seed):
    rng = np.random.default_rng(seed)
    sig = np.sqrt(np.log1p(0.25))
    ctx = np.maximum(256, np.round(np.exp(np.log(28100) - 0.5 * sig**2 + sig * rng.standard_normal(n)))).astype(np.int64)
    qry = np.maximum(1, np.round(np.exp(np.log(28) - 0.5 * sig**2 + sig * rng.standard_normal(n)))).astype(np.int64)
    arr = np.cumsum(np.maximum(rng.exponential(1.0, n) / qps, 1e-6))
    hit = rng.choice([0.25, 0.5, 0.75, 1.0], n)
    return t.QueueArrays(n, id=np.arange(1, n + 1), arrival=arr, context_tokens=ctx, query_tokens=qry,
                         cache_hit_ratio=hit, flags=np.zeros(n, np.uint8))


def des(po, q, cfg, policy, models):
    ttft = np.zeros(q.n)
    mean = C.c_double()
    st = po.ref().ref_run_simulation(q.n, C.byref(po.queue_struct(q)), C.byref(po.cluster_struct(cfg)), int(policy),
                                     (C.c_double * 4)(models.load.slope, models.load.intercept, models.comp.slope,
                                                      models.comp.intercept), 0, ttft.ctypes.data, C.byref(mean))
    if st != 0:
        raise RuntimeError(po.ref().ref_last_error().decode())
    return ttft


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=80)
    ap.add_argument("--qps", type=float, default=18.0)
    ap.add_argument("--compute-per-token", type=float, default=4e-6)
    ap.add_argument("--l1-gib", type=int, default=40)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    import pyoracle as po

    shape = ingest.LLAMA31_8B
    q = loogle_stream(args.n, args.qps, args.seed)
    bpt = t.kv_bytes_per_token(32, 8, 128, 2)
    plans = [int(np.floor(q.context_tokens[i] * q.cache_hit_ratio[i] / 256)) for i in range(q.n)]
    n_slots = 512
    pool = ingest.ChunkPool(shape, n_slots)
    pool.fill_synthetic(1)
    rng = np.random.default_rng(args.seed + 1)
    slots = []
    for nb in plans:
        s0 = int(rng.integers(0, n_slots - nb + 1))
        slots.append(list(range(s0, s0 + nb)))
    num_pages = (args.l1_gib << 30) // shape.page_bytes
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=q.n + 1, max_chunks=max(plans) + 1)
    stage = LoadStage(l1, pool)

    # calibrate the ingest rate on this box (batch stage, whole plan set, no prefill)
    base_cfg = t.ClusterConfig(bytes_per_token=bpt, compute_per_token=args.compute_per_token)
    stage.run(q, slots, base_cfg)
    r = stage.run(q, slots, base_cfg)
    rate = r.stats["bytes"] / (r.requests["resident_ms"].max() * 1e-3)
    cfg = t.ClusterConfig(bytes_per_token=bpt, network_bandwidth=rate, pcie_bandwidth=1e18, transfer_base_latency=0.0,
                          l1_capacity=num_pages * shape.page_bytes, l2_capacity=10**15, compute_base=2e-3,
                          compute_per_token=args.compute_per_token)
    models = t.cost_models_from_config(cfg)
    # deadlines: factor x solo TTFT in an empty system (workload.cpp:101-131), via the DES
    solo = np.array([des(po, t.QueueArrays(1, **{k: getattr(q, k)[i:i + 1].copy() for k, _ in t.QueueArrays.FIELDS}),
                         cfg, t.PolicyKind.Fifo, models)[0] for i in range(q.n)])
    factor = np.random.default_rng(args.seed + 2).choice([2.0, 4.0, 8.0], q.n)
    q.deadline[:] = q.arrival + factor * solo
    q.flags[:] = 1
    out = {"workload": f"{q.n} LooGLE-like requests (ctx mean 28100 cv .5, hit .25-1.0), Poisson {args.qps} QPS, "
                       f"Llama-3.1-8B KV, L1 {args.l1_gib} GiB, prefill {args.compute_per_token:g} s/token + 2 ms",
           "ingest_GBps_calibrated": rate / 1e9, "policies": {}}
    for pol in t.PolicyKind:
        res = stage.run_online(q, slots, cfg, models=models, policy=pol)
        req = res.requests
        ttft = (req["done_ms"] - req["arrival_ms"]) * 1e-3
        sim = des(po, q, cfg, pol, models)
        dl = q.deadline - q.arrival
        out["policies"][t.policy_name(pol)] = {
            "real_mean_ttft_s": float(ttft.mean()), "sim_mean_ttft_s": float(sim.mean()),
            "real_slo_attainment": float((ttft <= dl).mean()), "sim_slo_attainment": float((sim <= dl).mean()),
            "mean_abs_rel_err": float(np.mean(np.abs(ttft - sim) / sim)),
            "deferred_chunks": int(res.stats["deferred_chunks"])}
        print(json.dumps({t.policy_name(pol): out["policies"][t.policy_name(pol)]}), file=sys.stderr, flush=True)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
