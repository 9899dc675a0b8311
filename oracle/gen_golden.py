"""Generate tests/golden/* from the compiled reference (oracle/_ref) -- TEST INFRASTRUCTURE.

Run in the build container (where /root/reference exists):  python oracle/gen_golden.py
The fixtures travel with the repo so the GPU box (which has no /root/reference) can check the
CUDA path against the reference's own outputs.

  ref_queue.npz     a 1500-request generate_workload(loogle) queue (+ deadlines, measured-cost
                    rows) and, per policy, the reference's t_load/t_comp/primary (bit patterns)
                    and std::sort order under PriorityKey::operator<
  ref_plan.npz      make_request_state plans for edge-case (ctx, query, hit) triples
  ref_ledger.npz    a random TierLedger request/release script and the reference's decisions
  ref_misc.json     kv_bytes_per_token, cost_models_from_config, config_fingerprint values
  hash_frozen.npz   frozen prefix-hash vectors of the restatement (definition regression)
  ref_workload.npz  generate_workload streams (builtin + custom profiles, fixed and uniform hit
                    sources) and assign_slos deadlines, for the product's own generator

  python oracle/gen_golden.py --only workload   regenerates ref_workload.npz alone
"""
from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import pyoracle as po  # noqa: E402

GOLD = ROOT / "tests" / "golden"


class Q:
    """Minimal QueueArrays stand-in (numpy SoA) so the oracle does not import the product."""

    NAMES = ("id", "arrival", "context_tokens", "query_tokens", "cache_hit_ratio", "flags", "deadline",
             "measured_t_load", "measured_t_comp")

    def __init__(self, **a):
        for k in self.NAMES:
            setattr(self, k, a[k])
        self.n = len(self.id)


class Cfg:
    def __init__(self, **kw):
        d = dict(network_bandwidth=50e9, pcie_bandwidth=64e9, transfer_base_latency=10e-6,
                 l1_capacity=80_000_000_000, l2_capacity=128_000_000_000, bytes_per_token=131072,
                 block_size_tokens=256, compute_base=2e-3, compute_per_token=4e-5, compute_quadratic=0.0,
                 allocation_mode=0, control_mode=1)
        d.update(kw)
        self.__dict__.update(d)


def ref_models(cfg):
    m = (C.c_double * 4)()
    po.ref().ref_cost_models_from_config(C.byref(po.cluster_struct(cfg)), m)
    return list(m)


def make_queue(n=1500, seed=7):
    ids, arr, ctx, qry, hit = po.generate_workload("loogle", n, seed, qps=2.0,
                                                   hit_choices=[0.0, 0.25, 0.5, 0.75, 0.9, 1.0])
    rng = np.random.default_rng(seed)
    flags = np.full(n, 1, np.uint8)  # every request has a deadline
    deadline = arr + rng.choice([2.0, 4.0, 8.0], n) * (0.05 + ctx * 4e-5)
    ml, mc = np.zeros(n), np.zeros(n)
    meas = rng.random(n) < 0.05  # 5% replay measured costs verbatim (cost_model.cpp:58-59)
    flags[meas] |= 2
    ml[meas] = np.round(rng.random(meas.sum()) * 0.5, 3)
    mc[meas] = np.round(rng.random(meas.sum()) * 0.05, 3)
    # ties: duplicate arrivals and keys so the (arrival, id) tie-breaks matter
    arr[10:20] = arr[10]
    ctx[30:40] = ctx[30]
    hit[30:40] = hit[30]
    qry[30:40] = qry[30]
    return Q(id=ids, arrival=arr, context_tokens=ctx, query_tokens=qry, cache_hit_ratio=hit, flags=flags,
             deadline=deadline, measured_t_load=ml, measured_t_comp=mc)


def main():
    assert po.ref() is not None, "compiled reference required (make -C oracle ref)"
    GOLD.mkdir(parents=True, exist_ok=True)
    r = po.ref()

    # ---- queue + scores + order -----------------------------------------------------------
    q = make_queue()
    out = {k: getattr(q, k) for k in Q.NAMES}
    for cname, cfg in (("default", Cfg()), ("quad", Cfg(compute_quadratic=1e-9, block_size_tokens=128))):
        models = ref_models(cfg)
        out[f"{cname}_models"] = np.array(models)
        for pol in range(5):
            st, err, tl, tc, pr = po.score_queue(q, pol, models, cfg, which="ref")
            assert st == 0, r.ref_last_error()
            out[f"{cname}_p{pol}_t_load"] = tl.view(np.uint64)
            out[f"{cname}_p{pol}_t_comp"] = tc.view(np.uint64)
            out[f"{cname}_p{pol}_primary"] = pr.view(np.uint64)
            out[f"{cname}_p{pol}_order"] = po.ref_sort_order(q, pol, models, cfg)
    # drain order (pick_next) of the first 300 under each policy: pins sort == drain
    q300 = Q(**{k: np.ascontiguousarray(getattr(q, k)[:300]) for k in Q.NAMES})
    for pol in range(5):
        out[f"drain300_p{pol}"] = po.ref_drain_order(q300, pol, ref_models(Cfg()), Cfg())
    np.savez_compressed(GOLD / "ref_queue.npz", **out)

    # ---- plans -----------------------------------------------------------------------------
    cases = []
    for ctx in (0, 1, 255, 256, 257, 512, 28100, 32768, 131072, 1_000_003):
        for hit in (0.0, 0.1, 0.25, 0.5, 0.9, 0.999, 1.0):
            for block in (1, 16, 256):
                cases.append((ctx, 10, hit, block))
    plan = np.zeros((len(cases), 5), np.int64)
    for i, (ctx, qq, hit, block) in enumerate(cases):
        qi = Q(id=np.array([1], np.int64), arrival=np.zeros(1), context_tokens=np.array([ctx], np.int64),
               query_tokens=np.array([qq], np.int64), cache_hit_ratio=np.array([hit]), flags=np.zeros(1, np.uint8),
               deadline=np.zeros(1), measured_t_load=np.zeros(1), measured_t_comp=np.zeros(1))
        vals = [C.c_int64() for _ in range(5)]
        st = r.ref_block_plan(C.byref(po.queue_struct(qi)), 0, C.byref(po.cluster_struct(Cfg(block_size_tokens=block))),
                              *[C.byref(v) for v in vals])
        assert st == 0
        plan[i] = [v.value for v in vals]
    np.savez_compressed(GOLD / "ref_plan.npz", cases=np.array(cases, dtype=np.float64), plan=plan)

    # ---- ledger script -----------------------------------------------------------------------
    rng = np.random.default_rng(3)
    cap = 1000
    led = r.ref_ledger_new(2, cap)
    ops, results = [], []
    live = []
    for step in range(4000):
        if live and rng.random() < 0.45:
            b = int(live.pop(int(rng.integers(len(live)))))
            rid = (C.c_int64 * 64)()
            blk = (C.c_int32 * 64)()
            by = (C.c_int64 * 64)()
            n = C.c_int64()
            st = r.ref_ledger_release(led, b, rid, blk, by, 64, C.byref(n))
            assert st == 0
            grants = [(rid[i], blk[i], by[i]) for i in range(n.value)]
            live.extend(g[2] for g in grants)
            ops.append((1, b, 0, 0))
            results.append((st, n.value, r.ref_ledger_reserved(led), r.ref_ledger_deferred(led),
                            json.dumps(grants)))
        else:
            b = int(rng.integers(1, 300))
            g = C.c_int()
            st = r.ref_ledger_request(led, step, step % 7, b, C.byref(g))
            if st == 0 and g.value:
                live.append(b)
            ops.append((0, b, step, step % 7))
            results.append((st, g.value, r.ref_ledger_reserved(led), r.ref_ledger_deferred(led), "[]"))
    r.ref_ledger_free(led)
    np.savez_compressed(GOLD / "ref_ledger.npz", capacity=cap, ops=np.array(ops, np.int64),
                        res=np.array([x[:4] for x in results], np.int64),
                        grants=np.array([x[4] for x in results]))

    # ---- misc scalars ------------------------------------------------------------------------
    misc = {"kv_bytes_per_token": {}, "models": {}, "fingerprint": []}
    for name, shape in (("llama31_8b", (32, 8, 128, 2)), ("qwen25_32b", (64, 8, 128, 2)),
                        ("llama3_70b", (80, 8, 128, 2))):
        v = C.c_int64()
        assert r.ref_kv_bytes_per_token(*shape, C.byref(v)) == 0
        misc["kv_bytes_per_token"][name] = v.value
    misc["models"]["default"] = [float(x).hex() for x in ref_models(Cfg())]
    for cfg, pol, seed in ((Cfg(), 0, 0), (Cfg(pcie_bandwidth=55.6e9), 4, 7), (Cfg(control_mode=0), 2, 123456789)):
        h = r.ref_config_fingerprint(C.byref(po.cluster_struct(cfg)), pol, seed)
        misc["fingerprint"].append({"cfg": cfg.__dict__, "policy": pol, "seed": seed, "hash": str(h)})
    (GOLD / "ref_misc.json").write_text(json.dumps(misc, indent=1))

    # ---- frozen prefix-hash vectors (restatement; the reference has no prefix hasher) --------
    offs = np.array([0, 0, 255, 511, 1791, 1791 + 4096, 1791 + 4096 + 1300], np.int64)
    doc = np.array([0, 0, 1, 0, 2, 0], np.int64)
    shared = np.array([0, 255, 256, 1280, 4096, 768], np.int64)
    toks = po.gen_tokens(42, offs, doc, shared)
    hashes = po.hash_prefix_chunks(offs, toks)
    np.savez_compressed(GOLD / "hash_frozen.npz", offsets=offs, doc=doc, shared=shared, tokens=toks,
                        hashes=hashes, synth=po.synth_fill(11, 12345, 64))
    print("golden fixtures written to", GOLD)


WORKLOAD_CASES = [
    # (profile, ctx_mean, ctx_cv, q_mean, q_cv, count, qps, seed, hit_kind, hit_fixed, choices)
    ("loogle", 0, 0, 0, 0, 0, 1.0, 0, 0, 1.0, []),
    ("loogle", 0, 0, 0, 0, 2000, 18.0, 7, 1, 0.0, [0.25, 0.5, 0.75, 1.0]),
    ("icl", 0, 0, 0, 0, 500, 3.5, 123456789, 0, 0.9, []),
    ("code", 0, 0, 0, 0, 300, 0.25, 2**63 + 11, 1, 0.0, [0.0, 1.0]),
    ("custom", 24000.0, 1.0, 28.0, 0.5, 1000, 8.0, 3, 1, 0.0, [0.25, 0.5, 0.75, 0.9, 1.0]),
    ("custom", 5000.0, 0.0, 10.0, 0.0, 50, 1e9, 5, 0, 0.5, []),
]


def gen_workload():
    r = po.ref()
    out = {}
    for k, (prof, cm, cc, qm, qc, count, qps, seed, hk, hf, ch) in enumerate(WORKLOAD_CASES):
        n = count or 120
        ids, arr, ctx, qry, hit = po.generate_workload(prof, n, seed, qps=qps, hit_fixed=hf,
                                                       hit_choices=ch if hk else None, ctx_mean=cm, ctx_cv=cc,
                                                       q_mean=qm, q_cv=qc)
        q = Q(id=ids, arrival=arr, context_tokens=ctx, query_tokens=qry, cache_hit_ratio=hit,
              flags=np.zeros(n, np.uint8), deadline=np.zeros(n), measured_t_load=np.zeros(n),
              measured_t_comp=np.zeros(n))
        if k == 1:  # some measured-cost rows for the solo-baseline replay path
            q.flags[::7] = 2
            q.measured_t_load[::7] = np.linspace(0.0, 0.3, len(q.flags[::7]))
            q.measured_t_comp[::7] = 0.01
        cfg = Cfg(bytes_per_token=262144, l1_capacity=10**13, l2_capacity=10**13) if k == 4 else Cfg()
        dl = np.empty(n)
        fac = np.array([2.0, 4.0, 8.0])
        st = r.ref_assign_slos(n, C.byref(po.queue_struct(q)), C.byref(po.cluster_struct(cfg)),
                               (C.c_double * 4)(*ref_models(cfg)), fac.ctypes.data, 3, seed, dl.ctypes.data)
        assert st == 0, r.ref_last_error()
        for name in ("id", "arrival", "context_tokens", "query_tokens", "cache_hit_ratio", "flags",
                     "measured_t_load", "measured_t_comp"):
            out[f"c{k}_{name}"] = getattr(q, name)
        out[f"c{k}_deadline"] = dl
        out[f"c{k}_cfg"] = np.array([cfg.bytes_per_token, cfg.l1_capacity, cfg.l2_capacity])
    np.savez_compressed(GOLD / "ref_workload.npz", **out)
    print("wrote", GOLD / "ref_workload.npz")


if __name__ == "__main__":
    if sys.argv[1:] == ["--only", "workload"]:
        gen_workload()
    else:
        main()
        gen_workload()
