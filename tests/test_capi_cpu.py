"""The C-ABI library on CPU: loads, exports every declared symbol, and its host-side planning /
ledger logic reproduces the reference goldens (no device compute is called here)."""
import ctypes as C
import json
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2603_21257_b200 as pkg
from paper_2603_21257_b200 import _capi
from paper_2603_21257_b200 import tiersim as t

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    src = (ROOT / "include" / "tsb_capi.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tsb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) > 50
    missing = [n for n in names if not hasattr(_capi.lib, n)]
    assert not missing, missing


def test_library_exports_nothing_undeclared():
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert exported == set(declared_functions())


def test_built_for_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_version_and_status_strings():
    assert b"sm_100a" in _capi.lib.tsb_version()
    with pytest.raises(t.ValidationError, match="kv_bytes_per_token: all arguments must be >= 1"):
        t.kv_bytes_per_token(32, 0, 128, 2)


def test_kv_bytes_per_token_goldens(golden):
    misc = json.loads(golden("ref_misc.json"))
    assert t.kv_bytes_per_token(32, 8, 128, 2) == misc["kv_bytes_per_token"]["llama31_8b"] == 131072
    assert t.kv_bytes_per_token(64, 8, 128, 2) == misc["kv_bytes_per_token"]["qwen25_32b"]
    assert t.kv_bytes_per_token(80, 8, 128, 2) == misc["kv_bytes_per_token"]["llama3_70b"]


def test_config_fingerprint_matches_reference_golden(golden):
    """tsb_config_fingerprint == the compiled reference's config_fingerprint (engine.cpp:516-534)
    on every golden (config, policy, seed), and it separates configs that differ in one field."""
    misc = json.loads(golden("ref_misc.json"))
    assert misc["fingerprint"]
    for fp in misc["fingerprint"]:
        cfg = dict(fp["cfg"])
        cfg["allocation_mode"] = t.AllocationMode(cfg["allocation_mode"])
        cfg["control_mode"] = t.ControlMode(cfg["control_mode"])
        assert t.config_fingerprint(t.ClusterConfig(**cfg), fp["policy"], int(fp["seed"])) == int(fp["hash"])
    base = t.ClusterConfig()
    seen = {t.config_fingerprint(base, 0, 1), t.config_fingerprint(base, 1, 1), t.config_fingerprint(base, 0, 2),
            t.config_fingerprint(t.ClusterConfig(compute_quadratic=1e-9), 0, 1),
            t.config_fingerprint(t.ClusterConfig(control_mode=t.ControlMode.Coupled), 0, 1)}
    assert len(seen) == 5


def test_block_plans_match_reference_golden(golden):
    g = golden("ref_plan.npz")
    for (ctx, qry, hit, block), (cached, comp, nb, btok, bbytes) in zip(g["cases"], g["plan"]):
        spec = t.RequestSpec(id=1, context_tokens=int(ctx), query_tokens=int(qry), cache_hit_ratio=float(hit))
        cfg = t.ClusterConfig(block_size_tokens=int(block))
        plan = t.derive_block_plan(spec, cfg)
        assert len(plan) == nb
        assert t.cached_token_count(spec, cfg) == cached
        assert t.compute_token_count(spec, cfg) == comp
        assert all(b.tokens == btok and b.bytes == bbytes for b in plan)
        assert [b.block_index for b in plan] == list(range(nb))


def test_reference_types_goldens():
    """test_types.cpp:24-77"""
    cfg = t.ClusterConfig()
    assert len(t.derive_block_plan(t.RequestSpec(id=1, context_tokens=512, query_tokens=10), cfg)) == 2
    spec = t.RequestSpec(id=1, context_tokens=28100, query_tokens=10)
    assert len(t.derive_block_plan(spec, cfg)) == 109 and t.cached_token_count(spec, cfg) == 27904
    assert t.derive_block_plan(t.RequestSpec(id=1, context_tokens=28100, cache_hit_ratio=0.0), cfg) == []
    with pytest.raises(t.ValidationError, match="cache_hit_ratio"):
        t.RequestSpec(id=3, context_tokens=10, cache_hit_ratio=1.5).validate()
    with pytest.raises(t.ValidationError, match="query_tokens"):
        t.RequestSpec(id=3, context_tokens=10, query_tokens=0).validate()
    with pytest.raises(t.ValidationError, match="deadline"):
        t.RequestSpec(id=3, arrival_time=2.0, deadline=1.0).validate()
    with pytest.raises(t.ValidationError, match="network_bandwidth"):
        t.ClusterConfig(network_bandwidth=0).validate()


def test_cost_model_goldens(golden):
    misc = json.loads(golden("ref_misc.json"))
    m = t.cost_models_from_config(t.ClusterConfig())
    assert [float(x).hex() for x in (m.load.slope, m.load.intercept, m.comp.slope, m.comp.intercept)] == \
        misc["models"]["default"]
    assert t.predict(t.LinearCostModel(1e-4, 0.1), 2610) == pytest.approx(0.361, rel=1e-12)
    cost = t.estimate_service_cost(t.RequestSpec(id=1, context_tokens=1000, query_tokens=10,
                                                 measured_cost=t.MeasuredCost(0.361, 0.019)),
                                   t.LinearCostModel(1e-5), t.LinearCostModel(1e-5), t.ClusterConfig())
    assert (cost.t_load, cost.t_comp) == (0.361, 0.019)
    fit = t.fit_linear([(0, 0.1), (1000, 0.2), (2000, 0.3)])
    assert fit.model.slope == pytest.approx(1e-4) and fit.model.intercept == pytest.approx(0.1)
    with pytest.raises(t.DegenerateFit):
        t.fit_linear([(5, 0.1), (5, 0.2)])
    f = t.fit_linear([(0, 0.5), (1000, 0.1)])
    assert f.model.slope == 0.0 and f.slope_clamped


@pytest.mark.parametrize("policy", range(5))
def test_scalar_host_cost_and_key_match_reference_bits(golden, policy):
    g = golden("ref_queue.npz")
    cfg = t.ClusterConfig()
    m = t.cost_models_from_config(cfg)
    q = t.QueueArrays(**{k: g[k] for k, _ in t.QueueArrays.FIELDS})
    qs = q.struct()
    for i in range(0, q.n, 7):
        a, b, p = C.c_double(), C.c_double(), C.c_double()
        t.check(_capi.lib.tsb_estimate_service_cost(C.byref(qs), i, m.array(), C.byref(cfg.struct()), C.byref(a), C.byref(b)))
        t.check(_capi.lib.tsb_priority_key(C.byref(qs), i, policy, a.value, b.value, C.byref(p)))
        assert np.float64(a.value).view(np.uint64) == g[f"default_p{policy}_t_load"][i]
        assert np.float64(b.value).view(np.uint64) == g[f"default_p{policy}_t_comp"][i]
        assert np.float64(p.value).view(np.uint64) == g[f"default_p{policy}_primary"][i]


def test_priority_key_missing_deadline_message():
    spec = t.RequestSpec(id=42, context_tokens=100)
    with pytest.raises(t.MissingDeadline, match="lstf: request 42 has no deadline"):
        t.priority_key(spec, t.PolicyKind.Lstf, t.ServiceCost())
    k = t.priority_key(spec, t.PolicyKind.SjfPt, t.ServiceCost())
    assert k.primary == 101.0 - 100.0 and (k.arrival, k.id) == (0.0, 42)


def test_policy_names_round_trip():
    for p in t.all_policies():
        assert t.policy_from_name(t.policy_name(p)) == p
    assert t.policy_from_name("sjf") is None


def test_ledger_reference_goldens():
    """test_engine.cpp:64-91 on the libtsb ledger (the object the L1 allocator runs)."""
    led = t.TierLedger(t.Tier.L1, 100)
    assert led.request(1, 0, 40) == t.TierLedger.Granted
    assert led.request(1, 1, 60) == t.TierLedger.Granted
    assert led.reserved() == 100
    led = t.TierLedger(t.Tier.L1, 100)
    assert led.request(1, 0, 90) == t.TierLedger.Granted
    assert led.request(2, 0, 20) == t.TierLedger.Deferred
    assert led.request(3, 0, 5) == t.TierLedger.Deferred
    assert led.deferred_count() == 2
    granted = led.release(20)
    assert [g.request_id for g in granted] == [2, 3] and led.reserved() == 95
    led = t.TierLedger(t.Tier.L2, 100)
    with pytest.raises(t.CapacityError, match="l2: reservation of 101 bytes exceeds capacity 100"):
        led.request(1, 0, 101)
    with pytest.raises(t.ValidationError):
        led.request(1, 0, 0)
    with pytest.raises(t.ValidationError):
        led.release(1)
    with pytest.raises(t.ValidationError):
        t.TierLedger(t.Tier.L1, 0)


def test_ledger_replays_reference_script(golden):
    g = golden("ref_ledger.npz")
    led = t.TierLedger(t.Tier.L1, int(g["capacity"]))
    for (op, b, rid, blk), (st, val, reserved, deferred), grants in zip(g["ops"], g["res"], g["grants"]):
        if op == 0:
            assert int(led.request(int(rid), int(blk), int(b)) == t.TierLedger.Granted) == val
        else:
            got = led.release(int(b))
            assert [[p.request_id, p.block_index, p.bytes] for p in got] == json.loads(str(grants))
        assert led.reserved() == reserved and led.deferred_count() == deferred
