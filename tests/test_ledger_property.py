"""Property test (CPU): the libtsb TierLedger (tsb_ledger_*, also the L1 allocator's decision
core) against the reference's own TierLedger compiled in place (oracle/_ref, engine.cpp:18-49),
step by step over random operation scripts: the same Granted/Deferred decisions, the same FIFO
grant lists on release, the same reserved / deferred counts, and the same error class (with the
reference's message text) for invalid sizes, over-capacity requests and over-release."""
import ctypes as C
import sys
from pathlib import Path

import pytest

hypothesis = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
from paper_2603_21257_b200 import tiersim as t  # noqa: E402

ORC_OK, ORC_VALIDATION, ORC_CAPACITY = 0, 1, 2
EXC = {ORC_VALIDATION: t.ValidationError, ORC_CAPACITY: t.CapacityError}

ops = st.lists(
    st.one_of(
        st.tuples(st.just("req"), st.integers(0, 7), st.integers(0, 40), st.integers(-5, 130)),
        st.tuples(st.just("rel"), st.just(0), st.just(0), st.integers(-5, 130)),
    ),
    min_size=1, max_size=60)


def _ref_release(ref, h, nbytes):
    cap = 256
    rid, blk, b = (C.c_int64 * cap)(), (C.c_int32 * cap)(), (C.c_int64 * cap)()
    n = C.c_int64()
    st_ = ref.ref_ledger_release(h, nbytes, rid, blk, b, cap, C.byref(n))
    return st_, [(rid[i], blk[i], b[i]) for i in range(n.value)]


@settings(max_examples=300, deadline=None)
@given(capacity=st.integers(1, 120), script=ops)
def test_ledger_matches_live_reference(ref_lib, capacity, script):
    ref = ref_lib
    h = ref.ref_ledger_new(int(t.Tier.L1), capacity)
    ours = t.TierLedger(t.Tier.L1, capacity)
    try:
        for op, rid, blk, nbytes in script:
            if op == "req":
                g = C.c_int()
                rst = ref.ref_ledger_request(h, rid, blk, nbytes, C.byref(g))
                if rst == ORC_OK:
                    got = ours.request(rid, blk, nbytes)
                    assert (got == t.TierLedger.Granted) == bool(g.value)
                else:
                    with pytest.raises(EXC[rst]) as e:
                        ours.request(rid, blk, nbytes)
                    assert str(e.value) == ref.ref_last_error().decode()
            else:
                rst, grants = _ref_release(ref, h, nbytes)
                if rst == ORC_OK:
                    got = ours.release(nbytes)
                    assert [(p.request_id, p.block_index, p.bytes) for p in got] == grants
                else:
                    with pytest.raises(EXC[rst]) as e:
                        ours.release(nbytes)
                    assert str(e.value) == ref.ref_last_error().decode()
            assert ours.reserved() == ref.ref_ledger_reserved(h)
            assert ours.deferred_count() == ref.ref_ledger_deferred(h)
    finally:
        ref.ref_ledger_free(h)


# --- the host scalar service-cost / priority-key path against the live reference --------------
finite = st.floats(min_value=-1e6, max_value=1e9, allow_nan=False, allow_infinity=False)
requests = st.fixed_dictionaries(dict(
    id=st.integers(-2**40, 2**40),
    arrival=st.floats(min_value=0.0, max_value=1e7, allow_nan=False),
    context_tokens=st.integers(0, 10_000_000),
    query_tokens=st.integers(0, 100_000),
    cache_hit_ratio=st.one_of(st.sampled_from([0.0, 1e-12, 0.1, 1 / 3, 0.5, 0.9, 1 - 1e-12, 1.0]),
                              st.floats(min_value=0.0, max_value=1.0)),
    flags=st.sampled_from([0, 1, 2, 3]),
    deadline=st.floats(min_value=0.0, max_value=1e7, allow_nan=False),
    measured_t_load=st.floats(min_value=0.0, max_value=1e3, allow_nan=False),
    measured_t_comp=st.floats(min_value=0.0, max_value=1e3, allow_nan=False),
))


@settings(max_examples=400, deadline=None)
@given(r=requests, quad=st.sampled_from([0.0, 3e-10, 1e-6]), block=st.sampled_from([1, 16, 256, 1000]),
       policy=st.integers(0, 4))
def test_scalar_cost_and_key_match_live_reference(ref_lib, r, quad, block, policy):
    import numpy as np
    import pyoracle as po

    q = t.QueueArrays(1, **{k: np.array([v]) for k, v in r.items()})
    cfg = t.ClusterConfig(compute_quadratic=quad, block_size_tokens=block)
    m = t.cost_models_from_config(cfg)
    models = [m.load.slope, m.load.intercept, m.comp.slope, m.comp.intercept]
    _, _, rtl, rtc, _ = po.score_queue(q, 0, models, cfg, which="ref")  # costs do not depend on the policy
    st_, _, _, _, rpr = po.score_queue(q, policy, models, cfg, which="ref")
    qs = q.struct()
    a, b, p = C.c_double(), C.c_double(), C.c_double()
    from paper_2603_21257_b200 import _capi

    t.check(_capi.lib.tsb_estimate_service_cost(C.byref(qs), 0, m.array(), C.byref(cfg.struct()), C.byref(a),
                                                C.byref(b)))
    assert np.float64(a.value).view(np.uint64) == rtl.view(np.uint64)[0]
    assert np.float64(b.value).view(np.uint64) == rtc.view(np.uint64)[0]
    rc = _capi.lib.tsb_priority_key(C.byref(qs), 0, policy, a.value, b.value, C.byref(p))
    if st_ == 0:
        assert rc == 0 and np.float64(p.value).view(np.uint64) == rpr.view(np.uint64)[0]
    else:
        assert rc != 0  # MissingDeadline for EDF / LSTF without a deadline, as in the reference
