"""The product's own request-stream generator and SLO assignment (tsb_generate_workload,
tsb_solo_baseline_ttft, tsb_assign_slos) against the reference's generate_workload / assign_slos
(workload.cpp:70-135): the committed fixtures from oracle/_ref, and the live compiled reference
when it is built here.  Host arithmetic only (no device calls)."""
import ctypes as C
import sys

import numpy as np
import pytest

from paper_2603_21257_b200 import tiersim as t

sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1] / "oracle"))
from gen_golden import WORKLOAD_CASES  # noqa: E402  (the case table the fixtures were made from)


def spec_of(case):
    prof, cm, cc, qm, qc, count, qps, seed, hk, hf, ch = case
    p = t.builtin_profile(prof) if prof != "custom" else t.DatasetProfile("custom", count, cm, cc, qm, qc)
    src = t.HitRatioSource.uniform_choice(ch) if hk else t.HitRatioSource.fixed(hf)
    return t.WorkloadSpec(p, qps=qps, count=count, hit_ratio_source=src, seed=seed)


def cfg_of(g, k):
    bpt, l1, l2 = (int(x) for x in g[f"c{k}_cfg"])
    return t.ClusterConfig(bytes_per_token=bpt, l1_capacity=l1, l2_capacity=l2)


@pytest.mark.parametrize("k", range(len(WORKLOAD_CASES)))
def test_generate_workload_matches_reference_fixture(golden, k):
    g = golden("ref_workload.npz")
    q = t.generate_queue(spec_of(WORKLOAD_CASES[k]))
    for name in ("id", "context_tokens", "query_tokens"):
        assert np.array_equal(getattr(q, name), g[f"c{k}_{name}"]), name
    for name in ("arrival", "cache_hit_ratio"):  # bit patterns, not a tolerance
        assert np.array_equal(getattr(q, name).view(np.uint64), g[f"c{k}_{name}"].view(np.uint64)), name


@pytest.mark.parametrize("k", range(len(WORKLOAD_CASES)))
def test_assign_slos_matches_reference_fixture(golden, k):
    g = golden("ref_workload.npz")
    n = len(g[f"c{k}_id"])
    q = t.QueueArrays(n, **{name: g[f"c{k}_{name}"] for name in ("id", "arrival", "context_tokens", "query_tokens",
                                                                  "cache_hit_ratio", "flags", "measured_t_load",
                                                                  "measured_t_comp")})
    seed = WORKLOAD_CASES[k][7]
    t.assign_slos_queue(q, cfg_of(g, k), [2.0, 4.0, 8.0], seed)
    assert np.array_equal(q.deadline.view(np.uint64), g[f"c{k}_deadline"].view(np.uint64))
    assert np.all(q.flags & 1)


def test_builtin_profiles_and_errors():
    p = t.builtin_profile("loogle")
    assert (p.num_requests, p.context_tokens_mean, p.query_tokens_mean) == (120, 28100.0, 28.0)
    assert t.builtin_profile("code").context_tokens_mean == 38300.0
    with pytest.raises(t.UnknownProfile, match="unknown dataset profile: nope"):
        t.builtin_profile("nope")
    with pytest.raises(t.ValidationError, match="workload: qps must be > 0"):
        t.generate_queue(t.WorkloadSpec(t.builtin_profile("icl"), qps=0.0))
    with pytest.raises(t.ValidationError, match="hit_ratio_source: uniform set must be non-empty"):
        t.generate_queue(t.WorkloadSpec(t.builtin_profile("icl"), hit_ratio_source=t.HitRatioSource.uniform_choice([])))
    with pytest.raises(t.ValidationError, match="hit_ratio_source: choices must be in"):
        t.generate_queue(t.WorkloadSpec(t.builtin_profile("icl"), hit_ratio_source=t.HitRatioSource.uniform_choice([1.5])))
    with pytest.raises(t.ValidationError, match="assign_slos: factors must be > 1"):
        t.assign_slos([t.RequestSpec(1, 0.0, 512, 1, 1.0)], t.ClusterConfig(), None, [1.0], 0)
    # the solo run refuses a request that can never be resident (engine.cpp:213-217)
    with pytest.raises(t.CapacityError, match="resident bytes can never fit"):
        t.solo_baseline_ttft(t.RequestSpec(5, 0.0, 700_000, 1, 1.0), t.ClusterConfig())


def test_solo_baseline_ttft_closed_form():
    cfg = t.ClusterConfig()
    # 0 blocks: compute only
    r0 = t.RequestSpec(1, 3.0, 100, 28, 0.0)
    assert t.solo_baseline_ttft(r0, cfg) == cfg.compute_base + cfg.compute_per_token * 128.0
    # measured cost replay: t_load + t_comp
    rm = t.RequestSpec(2, 0.0, 1000, 1, 1.0, measured_cost=t.MeasuredCost(0.25, 0.125))
    assert t.solo_baseline_ttft(rm, cfg) == 0.25 + 0.0 + 0.125


def test_live_reference_streams_and_slos(ref_lib, oracle):
    """Random specs beyond the fixtures, against the compiled reference directly."""
    rng = np.random.default_rng(11)
    for trial in range(25):
        n = int(rng.integers(1, 400))
        seed = int(rng.integers(0, 2**63))
        hk = int(rng.integers(0, 2))
        ch = list(np.round(rng.random(int(rng.integers(1, 6))), 3)) if hk else []
        cm, cc = float(rng.uniform(500, 60000)), float(rng.choice([0.0, 0.3, 1.0]))
        qps = float(rng.choice([0.5, 4.0, 100.0]))
        case = ("custom", cm, cc, 30.0, 0.5, n, qps, seed, hk, 0.75, ch)
        q = t.generate_queue(spec_of(case))
        ids, arr, ctx, qry, hit = oracle.generate_workload("custom", n, seed, qps=qps, hit_fixed=0.75,
                                                           hit_choices=ch if hk else None, ctx_mean=cm, ctx_cv=cc,
                                                           q_mean=30.0, q_cv=0.5)
        assert np.array_equal(q.context_tokens, ctx) and np.array_equal(q.query_tokens, qry)
        assert np.array_equal(q.arrival.view(np.uint64), arr.view(np.uint64))
        assert np.array_equal(q.cache_hit_ratio.view(np.uint64), hit.view(np.uint64))
        cfg = t.ClusterConfig(l1_capacity=10**13, l2_capacity=10**13, pcie_bandwidth=float(rng.uniform(20e9, 64e9)),
                              compute_quadratic=float(rng.choice([0.0, 1e-9])))
        t.assign_slos_queue(q, cfg, [1.5, 3.0], seed)
        dl = np.empty(n)
        m = t.cost_models_from_config(cfg)
        fac = np.array([1.5, 3.0])
        q.flags[:] = 0
        st = ref_lib.ref_assign_slos(n, C.byref(oracle.queue_struct(q)), C.byref(oracle.cluster_struct(cfg)),
                                     (C.c_double * 4)(m.load.slope, m.load.intercept, m.comp.slope, m.comp.intercept),
                                     fac.ctypes.data, 2, seed, dl.ctypes.data)
        assert st == 0
        assert np.array_equal(q.deadline.view(np.uint64), dl.view(np.uint64)), trial
