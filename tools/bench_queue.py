"""configs[4]: scheduler cost scoring + prefix hashing over a 100K-request synthetic queue.

GPU (K4+K5, K3) device-timed with CUDA events, beside the compiled reference (oracle/_ref:
estimate_service_cost + priority_key + std::sort, single-threaded as the reference is) and the
oracle hash restatement on all host cores.  Prints one JSON line.
"""
from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
from paper_2603_21257_b200 import hasher  # noqa: E402
from paper_2603_21257_b200 import tiersim as t  # noqa: E402
from paper_2603_21257_b200.scorer import BatchScorer, DeviceQueue  # noqa: E402


def loogle_queue(n, seed):
    """generate_workload(loogle, n, seed) -- the product's own generator, bit-identical to the
    reference's (workload.cpp:70-99) -- with assign_slos {2, 4, 8} deadlines (workload.cpp:117-135)."""
    q = t.generate_queue(t.WorkloadSpec(t.builtin_profile("loogle"), qps=1.0, count=n, seed=seed))
    return t.assign_slos_queue(q, t.ClusterConfig(l1_capacity=10**13, l2_capacity=10**13), [2.0, 4.0, 8.0], seed)


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


def main():
    n = 100_000
    q = loogle_queue(n, 0)
    cfg = t.ClusterConfig()
    m = t.cost_models_from_config(cfg)
    sc = BatchScorer(0)
    dq = DeviceQueue(q)
    out = sc.score_device(dq, t.PolicyKind.Lstf, m, cfg)
    res = {"workload": f"configs[4]: {n}-request LooGLE-like queue, scoring + order (5 policies) and prefix hashing"}
    gpu = {}
    for pol in t.PolicyKind:
        gpu[t.policy_name(pol)] = timed(lambda: sc.score_device(dq, pol, m, cfg, out=out, check_errors=False)) * 1e6
    res["gpu_score_order_us"] = gpu
    sc.score(q, t.PolicyKind.Lstf, m, cfg)  # first call sizes the pinned staging blocks
    t0 = time.perf_counter()
    for _ in range(10):
        sc.score(q, t.PolicyKind.Lstf, m, cfg)
    res["gpu_score_order_host_api_us"] = (time.perf_counter() - t0) / 10 * 1e6

    # CPU: the compiled reference (single-threaded, like the reference) when present
    import pyoracle as po

    mm = [m.load.slope, m.load.intercept, m.comp.slope, m.comp.intercept]
    if po.ref() is not None:
        t0 = time.perf_counter()
        st, err, tl, tc, pr = po.score_queue(q, int(t.PolicyKind.Lstf), mm, cfg, which="ref")
        t1 = time.perf_counter()
        order = po.ref_sort_order(q, int(t.PolicyKind.Lstf), mm, cfg)
        t2 = time.perf_counter()
        res["cpu_reference"] = {"kind": "reference", "cores": 1, "score_us": (t1 - t0) * 1e6,
                                "score_plus_sort_us": (t2 - t1) * 1e6,
                                "note": "estimate_service_cost + priority_key per request, then std::sort with "
                                        "PriorityKey::operator< (sort re-scores: it is the full order)"}
        gpu_order = sc.score(q, t.PolicyKind.Lstf, m, cfg)[3]
        res["order_equal_reference"] = bool(np.array_equal(gpu_order, order))

    # K3 over the queue's full contexts (token ids generated on device)
    lens = q.context_tokens
    offs = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=offs[1:])
    dev = torch.device("cuda")
    rng = np.random.default_rng(1)
    d_offs = torch.from_numpy(offs).to(dev)
    doc = torch.from_numpy(rng.integers(0, 1000, n)).to(dev)
    sh = torch.from_numpy(lens // 2).to(dev)
    tok = torch.empty(int(offs[-1]), dtype=torch.int32, device=dev)
    hasher.gen_tokens_device(0, d_offs, doc, sh, tok)
    coff = torch.from_numpy(hasher.chunk_offsets(offs)).to(dev)
    hout = torch.empty(int(coff[-1]), dtype=torch.int64, device=dev)
    secs = timed(lambda: hasher.hash_prefix_chunks_device(d_offs, tok, coff, hout), reps=10)
    nbytes = tok.numel() * 4 + hout.numel() * 8
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    res["hash"] = {"tokens": int(offs[-1]), "chunks": int(coff[-1]), "ms": secs * 1e3, "GBps": nbytes / secs / 1e9,
                   "hbm_frac": nbytes / secs / 1e9 / peak, "algorithmic_bytes": int(nbytes)}
    # K7: index every chunk hash of the queue (the L2 pool index), then look the queue up
    idx = hasher.PrefixIndex(capacity=4 * hout.numel())
    slots_t = torch.arange(hout.numel(), dtype=torch.int64, device=dev)
    ins_s = timed(lambda: idx.insert_device(hout, slots_t), reps=1, warm=0)
    m_out = torch.empty(n, dtype=torch.int64, device=dev)
    s_out = torch.empty_like(hout)
    look_s = timed(lambda: idx.lookup_device(coff, hout, s_out, m_out), reps=10)
    live, full = idx.stats()
    res["index"] = {"entries": live, "capacity": idx.capacity, "insert_ms": ins_s * 1e3, "lookup_ms": look_s * 1e3,
                    "lookups_per_s": hout.numel() / look_s, "all_matched": bool((m_out.cpu().numpy() ==
                                                                                np.diff(hasher.chunk_offsets(offs))).all())}
    # CPU hash_ref on a sample of 2000 requests, all host threads
    k = 2000
    sample_tok = tok[: int(offs[k])].cpu().numpy()
    thr = os.cpu_count() or 1
    t0 = time.perf_counter()
    href = po.hash_prefix_chunks(offs[: k + 1], sample_tok, threads=thr)
    cpu_s = time.perf_counter() - t0
    res["hash_cpu_port"] = {"kind": "port", "cores": thr, "sample_requests": k,
                            "GBps": (sample_tok.nbytes + href.nbytes) / cpu_s / 1e9}
    res["hash_sample_equal_port"] = bool(np.array_equal(hout[: len(href)].cpu().numpy().view(np.uint64), href))
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
