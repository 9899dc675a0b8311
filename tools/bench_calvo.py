"""CALVO's central comparison on B200, all three tiers real: coupled vs decoupled control x the
scheduling policies, against the reference DES of the same stream.

  * stream: the product's generate_workload (LooGLE profile, Poisson arrivals), hits from
    {0.25, 0.5, 0.75, 1.0}; deadlines from assign_slos {2, 4, 8} x solo TTFT on this box's
    calibrated config (workload.cpp:70-135);
  * L3: a host store of document chunks (requests share documents); the network hop L3 -> L2 is
    made by host copy threads paced to `network_bandwidth` (an RDMA-class link); L2: pinned slots
    under TierLedger(L2); L1: paged HBM under TierLedger(L1); L2 -> L1: the real ingest;
  * compute: K6 at a B200-like 4 us/token + 2 ms per request;
  * for every (control, policy): real mean / p90 TTFT and SLO attainment from
    tsb_stage_run_online, and the same from tiersim_ref::run_simulation configured with the same
    network pacing and the measured L2 -> L1 rate.  Prints one JSON line.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch  # noqa: F401  (CUDA context for the package)

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
from paper_2603_21257_b200 import ingest  # noqa: E402
from paper_2603_21257_b200 import tiersim as t  # noqa: E402
from paper_2603_21257_b200.stage import LoadStage  # noqa: E402


def des(po, q, cfg, policy):
    m = t.cost_models_from_config(cfg)
    ttft = np.zeros(q.n)
    mean = C.c_double()
    st = po.ref().ref_run_simulation(q.n, C.byref(po.queue_struct(q)), C.byref(po.cluster_struct(cfg)), int(policy),
                                     (C.c_double * 4)(m.load.slope, m.load.intercept, m.comp.slope, m.comp.intercept),
                                     0, ttft.ctypes.data, C.byref(mean))
    if st != 0:
        raise RuntimeError(po.ref().ref_last_error().decode())
    return ttft


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=60)
    ap.add_argument("--qps", type=float, default=6.0)
    ap.add_argument("--net-gbps", type=float, default=25.0)
    ap.add_argument("--l2-slots", type=int, default=320)
    ap.add_argument("--l1-gib", type=int, default=24)
    ap.add_argument("--compute-per-token", type=float, default=4e-6)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--consumer", choices=["k6", "real"], default="k6",
                    help="real: PagedPrefill (FlashInfer paged prefill + Llama-8B GEMMs) as the prefill hook; "
                         "the DES then uses T_comp fitted to a serial batch pass of the same consumer")
    args = ap.parse_args()
    import pyoracle as po

    shape = ingest.LLAMA31_8B
    bpt = t.kv_bytes_per_token(32, 8, 128, 2)
    q = t.generate_queue(t.WorkloadSpec(t.builtin_profile("loogle"), qps=args.qps, count=args.n, seed=args.seed,
                                        hit_ratio_source=t.HitRatioSource.uniform_choice([0.25, 0.5, 0.75, 1.0])))
    q.context_tokens[:] = np.minimum(q.context_tokens, 64 * 1024)
    plans = [int(np.floor(q.context_tokens[i] * q.cache_hit_ratio[i] / 256)) for i in range(q.n)]
    # L3: 6 documents of up to max-plan chunks; request i reads a prefix of document i % 6
    n_docs, doc_len = 6, max(plans) + 1
    l3 = ingest.ChunkPool(shape, n_docs * doc_len)
    l3.fill_synthetic(11)
    slots = [list(range((i % n_docs) * doc_len, (i % n_docs) * doc_len + nb)) for i, nb in enumerate(plans)]
    l2 = ingest.ChunkPool(shape, args.l2_slots)
    num_pages = (args.l1_gib << 30) // shape.page_bytes
    l1 = ingest.PagedKVCache(shape, num_pages, max_rows=q.n + 1, max_chunks=max(plans) + 1)
    stage = LoadStage(l1, l2)

    # the box's L2 -> L1 rate for these chunks (batch stage over the L2 pool, no network, no prefill)
    base = t.ClusterConfig(bytes_per_token=bpt, l1_capacity=num_pages * shape.page_bytes,
                           l2_capacity=args.l2_slots * shape.chunk_bytes, compute_base=2e-3,
                           compute_per_token=args.compute_per_token, network_bandwidth=args.net_gbps * 1e9)
    cal_slots = [[s % args.l2_slots for s in sl] for sl in slots]
    stage.run(q, cal_slots, base)
    r = stage.run(q, cal_slots, base)
    link = r.stats["bytes"] / (r.requests["resident_ms"].max() * 1e-3)
    comp_base, comp_tok, compute_desc = 2e-3, args.compute_per_token, f"K6 {args.compute_per_token:g} s/token + 2 ms"
    if args.consumer == "real":
        from paper_2603_21257_b200 import calibrate
        from paper_2603_21257_b200.consumer import PagedPrefill

        consumer = PagedPrefill(l1, q, base)
        stage.set_prefill_hook(consumer)
        stage.run(q, cal_slots, base, prefill=True)  # JIT + warm-up
        fit = t.fit_linear((x.tokens, x.seconds) for x in
                           calibrate.compute_samples(stage.run(q, cal_slots, base, prefill=True).requests))
        comp_base, comp_tok = fit.model.intercept, fit.model.slope
        compute_desc = (f"PagedPrefill (FlashInfer + Llama-3.1-8B GEMMs); DES T_comp fitted: {comp_tok:.3e} s/token + "
                        f"{comp_base * 1e3:.2f} ms")
    stage.set_l3(l3, copy_threads=8)
    box = t.ClusterConfig(bytes_per_token=bpt, l1_capacity=num_pages * shape.page_bytes,
                          l2_capacity=args.l2_slots * shape.chunk_bytes, compute_base=comp_base,
                          compute_per_token=comp_tok, network_bandwidth=args.net_gbps * 1e9,
                          pcie_bandwidth=link)
    t.assign_slos_queue(q, box, [2.0, 4.0, 8.0], 7)
    dl = q.deadline - q.arrival
    out = {"workload": f"{q.n} LooGLE-profile requests (generate_workload seed {args.seed}), {args.qps} QPS, hits "
                       "{0.25,0.5,0.75,1.0}, contexts capped at 64K, 6 shared documents in L3, Llama-3.1-8B KV",
           "tiers": {"l3_to_l2": f"host copy threads paced to {args.net_gbps} GB/s", "l2_slots": args.l2_slots,
                     "l1_gib": args.l1_gib, "l2_to_l1_measured_GBps": link / 1e9},
           "compute": compute_desc, "runs": {}}
    first = True
    for control in (t.ControlMode.Decoupled, t.ControlMode.Coupled):
        for pol in (t.PolicyKind.Fifo, t.PolicyKind.SjfCost, t.PolicyKind.Edf, t.PolicyKind.Lstf):
            cfg = t.ClusterConfig(**{**box.__dict__, "control_mode": control})
            res = stage.run_online(q, slots, cfg, policy=pol, pace_network=True, verify_seed=11 if first else 0)
            if first:
                assert res.stats["verify_mismatches"] == 0
                first = False
            req = res.requests
            ttft = (req["done_ms"] - req["arrival_ms"]) * 1e-3
            sim = des(po, q, cfg, pol)
            key = f"{'coupled' if control == t.ControlMode.Coupled else 'decoupled'}/{t.policy_name(pol)}"
            out["runs"][key] = {
                "real_mean_ttft_s": float(ttft.mean()), "real_p90_ttft_s": float(np.percentile(ttft, 90)),
                "real_slo_attainment": float((ttft <= dl).mean()),
                "sim_mean_ttft_s": float(sim.mean()), "sim_slo_attainment": float((sim <= dl).mean()),
                "per_request_mean_abs_rel_err": float(np.mean(np.abs(ttft - sim) / sim)),
                "net_blocks": int(res.stats["net_blocks"]), "l2_deferred": int(res.stats["l2_deferred"]),
                "l1_deferred": int(res.stats["deferred_chunks"])}
            print(json.dumps({key: out["runs"][key]}), file=sys.stderr, flush=True)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
