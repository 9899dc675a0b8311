"""Reference-shaped Python mirror of the kept tiersim API, over libtsb.so.

Names, argument meaning and error behaviour follow /root/reference/proj/core/include/tiersim/
(types.hpp, cost_model.hpp, scheduler.hpp, engine.hpp TierLedger, error.hpp) so that parity tests
read like the reference's own doctest suites.  Scalar planning helpers run as host arithmetic
inside libtsb.so; everything batched (scorer, order, hashing, ingest) runs on the GPU through
the C ABI -- there is no CPU fallback in this package.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _capi as capi
from ._capi import lib


# ---- error.hpp:13-71 -----------------------------------------------------------------------
class Error(RuntimeError):
    """tiersim::Error"""


class ValidationError(Error):
    pass


class DegenerateFit(Error):
    pass


class MissingDeadline(Error):
    pass


class CapacityError(Error):
    pass


class CudaError(Error):
    pass


class Unsupported(Error):
    pass


class UnknownProfile(Error):
    """error.hpp:43-47"""


_STATUS = {
    capi.TSB_VALIDATION: ValidationError,
    capi.TSB_CAPACITY: CapacityError,
    capi.TSB_MISSING_DEADLINE: MissingDeadline,
    capi.TSB_DEGENERATE_FIT: DegenerateFit,
    capi.TSB_CUDA: CudaError,
    capi.TSB_UNSUPPORTED: Unsupported,
    capi.TSB_UNKNOWN_PROFILE: UnknownProfile,
}


def check(status: int) -> None:
    if status != capi.TSB_OK:
        raise _STATUS.get(status, Error)(capi.last_error())


# ---- types.hpp -------------------------------------------------------------------------------
class Tier(enum.IntEnum):
    L3 = 0
    L2 = 1
    L1 = 2


class AllocationMode(enum.IntEnum):
    Proactive = 0
    Reactive = 1


class ControlMode(enum.IntEnum):
    Coupled = 0
    Decoupled = 1


@dataclass
class MeasuredCost:
    t_load: float = 0.0
    t_comp: float = 0.0


@dataclass
class RequestSpec:
    """types.hpp:52-64"""

    id: int = 0
    arrival_time: float = 0.0
    context_tokens: int = 0
    query_tokens: int = 1
    cache_hit_ratio: float = 1.0
    deadline: Optional[float] = None
    measured_cost: Optional[MeasuredCost] = None
    dataset_tag: str = ""

    def validate(self) -> None:
        q = QueueArrays.from_specs([self])
        check(lib.tsb_request_validate(C.byref(q.struct()), 0))


@dataclass
class ClusterConfig:
    """types.hpp:82-97 (same defaults)."""

    network_bandwidth: float = 50e9
    pcie_bandwidth: float = 64e9
    transfer_base_latency: float = 10e-6
    l1_capacity: int = 80_000_000_000
    l2_capacity: int = 128_000_000_000
    bytes_per_token: int = 131072
    block_size_tokens: int = 256
    compute_base: float = 2e-3
    compute_per_token: float = 4e-5
    compute_quadratic: float = 0.0
    allocation_mode: AllocationMode = AllocationMode.Proactive
    control_mode: ControlMode = ControlMode.Decoupled

    def struct(self) -> capi.Cluster:
        c = capi.Cluster()
        for name, _ in capi.Cluster._fields_:
            setattr(c, name, int(getattr(self, name)) if name.endswith("mode") else getattr(self, name))
        return c

    def validate(self) -> None:
        check(lib.tsb_cluster_validate(C.byref(self.struct())))


@dataclass
class KVBlock:
    """types.hpp:104-111"""

    request_id: int = 0
    block_index: int = 0
    tokens: int = 0
    bytes: int = 0
    residency: Tier = Tier.L3


class QueueArrays:
    """Struct-of-arrays RequestSpec queue (numpy, host) matching tsb_queue."""

    FIELDS = (
        ("id", np.int64),
        ("arrival", np.float64),
        ("context_tokens", np.int64),
        ("query_tokens", np.int64),
        ("cache_hit_ratio", np.float64),
        ("flags", np.uint8),
        ("deadline", np.float64),
        ("measured_t_load", np.float64),
        ("measured_t_comp", np.float64),
    )

    def __init__(self, n: int = 0, **arrays):
        for name, dt in self.FIELDS:
            a = arrays.get(name)
            setattr(self, name, np.ascontiguousarray(a, dtype=dt) if a is not None else np.zeros(n, dtype=dt))
        self.n = len(self.id)

    @classmethod
    def from_specs(cls, specs: Sequence[RequestSpec], costs: Optional[dict] = None) -> "QueueArrays":
        n = len(specs)
        q = cls(n)
        for i, s in enumerate(specs):
            q.id[i] = s.id
            q.arrival[i] = s.arrival_time
            q.context_tokens[i] = s.context_tokens
            q.query_tokens[i] = s.query_tokens
            q.cache_hit_ratio[i] = s.cache_hit_ratio
            fl = 0
            if s.deadline is not None:
                fl |= capi.HAS_DEADLINE
                q.deadline[i] = s.deadline
            mc = s.measured_cost
            if costs is not None:  # CostMap semantics (scheduler.cpp:82-83): missing id -> zero
                mc = costs.get(s.id, ServiceCost())
            if mc is not None:
                fl |= capi.HAS_MEASURED
                q.measured_t_load[i] = mc.t_load
                q.measured_t_comp[i] = mc.t_comp
            q.flags[i] = fl
        return q

    def struct(self) -> capi.Queue:
        s = capi.Queue()
        for name, _ in self.FIELDS:
            setattr(s, name, getattr(self, name).ctypes.data)
        return s


def _q1(spec: RequestSpec):
    q = QueueArrays.from_specs([spec])
    return q, q.struct()


def config_fingerprint(config: ClusterConfig, policy: int, seed: int) -> int:
    """engine.hpp:68-74 / engine.cpp:516-534: FNV-1a-64 of the config fields, policy and seed."""
    return int(lib.tsb_config_fingerprint(C.byref(config.struct()), int(policy), int(seed)))


def kv_bytes_per_token(layers: int, kv_heads: int, head_dim: int, dtype_bytes: int) -> int:
    out = C.c_int64()
    check(lib.tsb_kv_bytes_per_token(layers, kv_heads, head_dim, dtype_bytes, C.byref(out)))
    return out.value


def _plan(spec: RequestSpec, config: ClusterConfig):
    q, s = _q1(spec)
    vals = [C.c_int64() for _ in range(5)]
    check(lib.tsb_derive_block_plan(C.byref(s), 0, C.byref(config.struct()), *[C.byref(v) for v in vals]))
    return [v.value for v in vals]


def cached_token_count(spec: RequestSpec, config: ClusterConfig) -> int:
    return _plan(spec, config)[0]


def compute_token_count(spec: RequestSpec, config: ClusterConfig) -> int:
    return _plan(spec, config)[1]


def derive_block_plan(spec: RequestSpec, config: ClusterConfig) -> list[KVBlock]:
    cached, _, n, tokens, nbytes = _plan(spec, config)
    return [KVBlock(spec.id, i, tokens, nbytes) for i in range(n)]


# ---- cost_model.hpp --------------------------------------------------------------------------
@dataclass
class LinearCostModel:
    slope: float = 0.0
    intercept: float = 0.0


@dataclass
class LinearFit:
    model: LinearCostModel
    slope_clamped: bool = False
    intercept_clamped: bool = False


@dataclass
class ServiceCost:
    t_load: float = 0.0
    t_comp: float = 0.0

    def total(self) -> float:
        return self.t_load + self.t_comp


@dataclass
class CostModelPair:
    load: LinearCostModel = field(default_factory=LinearCostModel)
    comp: LinearCostModel = field(default_factory=LinearCostModel)

    def array(self):
        return (C.c_double * 4)(self.load.slope, self.load.intercept, self.comp.slope, self.comp.intercept)


def cost_models_from_config(config: ClusterConfig) -> CostModelPair:
    m = (C.c_double * 4)()
    lib.tsb_cost_models_from_config(C.byref(config.struct()), m)
    return CostModelPair(LinearCostModel(m[0], m[1]), LinearCostModel(m[2], m[3]))


def predict(model: LinearCostModel, tokens: int) -> float:
    return lib.tsb_predict(model.slope, model.intercept, int(tokens))


def fit_linear(samples: Iterable) -> LinearFit:
    samples = list(samples)
    tok = np.array([s[0] for s in samples], dtype=np.int64)
    sec = np.array([s[1] for s in samples], dtype=np.float64)
    a, b = C.c_double(), C.c_double()
    ca, cb = C.c_int(), C.c_int()
    check(lib.tsb_fit_linear(len(samples), tok.ctypes.data, sec.ctypes.data, C.byref(a), C.byref(b), C.byref(ca), C.byref(cb)))
    return LinearFit(LinearCostModel(a.value, b.value), bool(ca.value), bool(cb.value))


@dataclass
class TokenSample:
    """cost_model.hpp TokenSample: one measured (tokens, seconds) point."""

    tokens: int
    seconds: float


def read_samples_csv(path) -> list[TokenSample]:
    """cost_model.cpp:105-123: two columns (tokens, seconds) split on ',', ';', tab or spaces;
    '#' comments and blank lines skipped; a non-numeric FIRST line is a header; any later
    non-numeric line raises Error("read_samples_csv: malformed line in <path>: <line>")."""
    try:
        text = open(path).read()
    except OSError:
        raise Error(f"read_samples_csv: cannot open {path}") from None
    out, first = [], True
    for line in text.split("\n"):
        if not line or line[0] == "#":
            continue
        parts = line.replace(",", " ").replace(";", " ").replace("\t", " ").split()
        try:
            tokens, seconds = float(parts[0]), float(parts[1])
        except (IndexError, ValueError):
            if not first:
                raise Error(f"read_samples_csv: malformed line in {path}: {line}") from None
            first = False
            continue
        out.append(TokenSample(int(tokens), seconds))
        first = False
    return out


def write_samples_csv(path, samples, header: str = "tokens,seconds") -> None:
    """The file read_samples_csv reads: a header, then one 'tokens,seconds' row per sample
    (seconds printed with 17 significant digits, so the fit sees the measured doubles)."""
    with open(path, "w") as f:
        f.write(header + "\n")
        for s in samples:
            tok, sec = (s.tokens, s.seconds) if isinstance(s, TokenSample) else s
            f.write(f"{int(tok)},{float(sec):.17g}\n")


def estimate_service_cost(spec: RequestSpec, load_model: LinearCostModel, comp_model: LinearCostModel,
                          config: ClusterConfig) -> ServiceCost:
    q, s = _q1(spec)
    m = CostModelPair(load_model, comp_model).array()
    a, b = C.c_double(), C.c_double()
    check(lib.tsb_estimate_service_cost(C.byref(s), 0, m, C.byref(config.struct()), C.byref(a), C.byref(b)))
    return ServiceCost(a.value, b.value)


# ---- scheduler.hpp ---------------------------------------------------------------------------
class PolicyKind(enum.IntEnum):
    Fifo = 0
    SjfPt = 1
    SjfCost = 2
    Edf = 3
    Lstf = 4


_POLICY_NAMES = {"fifo": PolicyKind.Fifo, "sjf-pt": PolicyKind.SjfPt, "sjf-cost": PolicyKind.SjfCost,
                 "edf": PolicyKind.Edf, "lstf": PolicyKind.Lstf}


def policy_from_name(name: str) -> Optional[PolicyKind]:
    return _POLICY_NAMES.get(name)


def policy_name(policy: PolicyKind) -> str:
    return {v: k for k, v in _POLICY_NAMES.items()}[PolicyKind(policy)]


def all_policies() -> list[PolicyKind]:
    return list(PolicyKind)


@dataclass(frozen=True, order=False)
class PriorityKey:
    primary: float = 0.0
    arrival: float = 0.0
    id: int = 0

    def __lt__(self, other: "PriorityKey") -> bool:  # scheduler.hpp:38-42
        if self.primary != other.primary:
            return self.primary < other.primary
        if self.arrival != other.arrival:
            return self.arrival < other.arrival
        return self.id < other.id


def prefill_token_estimate(spec: RequestSpec) -> float:
    q, s = _q1(spec)
    out = C.c_double()
    check(lib.tsb_priority_key(C.byref(s), 0, int(PolicyKind.SjfPt), 0.0, 0.0, C.byref(out)))
    return out.value


def priority_key(spec: RequestSpec, policy: PolicyKind, cost: ServiceCost, now: float = 0.0) -> PriorityKey:
    q, s = _q1(spec)
    out = C.c_double()
    check(lib.tsb_priority_key(C.byref(s), 0, int(policy), cost.t_load, cost.t_comp, C.byref(out)))
    return PriorityKey(out.value, spec.arrival_time, spec.id)


# The batched GPU scorer (K4+K5) backs the queue operations below.
_default_scorer = None


def default_scorer():
    global _default_scorer
    if _default_scorer is None:
        from .scorer import BatchScorer

        _default_scorer = BatchScorer(device=0)
    return _default_scorer


def best_request_index(queue: Sequence[RequestSpec], policy: PolicyKind, costs: dict, now: float = 0.0):
    """scheduler.cpp:75-91 -- on the GPU: order[0] of the batched scorer with CostMap costs."""
    if not queue:
        return None
    order = default_scorer().order_specs(queue, policy, costs=costs)
    return int(order[0])


def pick_next(queue: list, policy: PolicyKind, costs: dict, now: float = 0.0):
    """scheduler.cpp:93-100: removes and returns the minimum-key request (None when empty)."""
    idx = best_request_index(queue, policy, costs, now)
    if idx is None:
        return None
    return queue.pop(idx)


def schedule_order(queue: Sequence[RequestSpec], policy: PolicyKind, costs: Optional[dict] = None,
                   models: Optional[CostModelPair] = None, config: Optional[ClusterConfig] = None) -> list[int]:
    """The full pick_next drain of a fixed queue as one GPU sort: returns request ids in pick order."""
    order = default_scorer().order_specs(queue, policy, costs=costs, models=models, config=config)
    return [queue[int(i)].id for i in order]


# ---- workload.hpp ----------------------------------------------------------------------------
@dataclass
class DatasetProfile:
    """workload.hpp:19-28"""

    name: str = ""
    num_requests: int = 0
    context_tokens_mean: float = 0.0
    context_tokens_cv: float = 0.5
    query_tokens_mean: float = 0.0
    query_tokens_cv: float = 0.5


def builtin_profile(name: str) -> DatasetProfile:
    """workload.cpp:31-36; raises UnknownProfile."""
    w = capi.WorkloadSpec()
    check(lib.tsb_builtin_profile(name.encode(), C.byref(w)))
    return DatasetProfile(name, w.num_requests, w.context_tokens_mean, w.context_tokens_cv, w.query_tokens_mean,
                          w.query_tokens_cv)


@dataclass
class HitRatioSource:
    """workload.hpp:33-45: a fixed value, or a uniform pick from `choices`."""

    fixed_value: Optional[float] = 1.0
    choices: Optional[Sequence[float]] = None

    @staticmethod
    def fixed(v: float) -> "HitRatioSource":
        return HitRatioSource(v, None)

    @staticmethod
    def uniform_choice(values: Sequence[float]) -> "HitRatioSource":
        return HitRatioSource(None, list(values))


@dataclass
class WorkloadSpec:
    """workload.hpp:55-68"""

    profile: DatasetProfile = field(default_factory=DatasetProfile)
    qps: float = 1.0
    count: int = 0
    hit_ratio_source: HitRatioSource = field(default_factory=HitRatioSource)
    seed: int = 0

    def _struct(self):
        w = capi.WorkloadSpec()
        p = self.profile
        w.num_requests, w.context_tokens_mean, w.context_tokens_cv = p.num_requests, p.context_tokens_mean, p.context_tokens_cv
        w.query_tokens_mean, w.query_tokens_cv = p.query_tokens_mean, p.query_tokens_cv
        w.qps, w.count, w.seed = self.qps, self.count, self.seed
        h = self.hit_ratio_source
        keep = None
        if h.choices is None:
            w.hit_kind, w.hit_fixed = 0, h.fixed_value
        else:
            keep = np.ascontiguousarray(h.choices, np.float64)
            w.hit_kind, w.hit_choices, w.n_hit_choices = 1, keep.ctypes.data, len(keep)
        return w, keep

    def effective_count(self) -> int:
        w, _ = self._struct()
        return lib.tsb_workload_count(C.byref(w))


def generate_queue(spec: WorkloadSpec) -> QueueArrays:
    """generate_workload (workload.cpp:70-99) as a struct-of-arrays queue (no deadlines)."""
    w, keep = spec._struct()
    check(lib.tsb_workload_validate(C.byref(w)))
    n = lib.tsb_workload_count(C.byref(w))
    q = QueueArrays(n)
    got = C.c_int64()
    check(lib.tsb_generate_workload(C.byref(w), n, q.id.ctypes.data, q.arrival.ctypes.data,
                                    q.context_tokens.ctypes.data, q.query_tokens.ctypes.data,
                                    q.cache_hit_ratio.ctypes.data, C.byref(got)))
    del keep
    return q


def generate_workload(spec: WorkloadSpec) -> list[RequestSpec]:
    """workload.cpp:70-99: the reference's RequestSpec stream, bit for bit."""
    q = generate_queue(spec)
    return [RequestSpec(int(q.id[i]), float(q.arrival[i]), int(q.context_tokens[i]), int(q.query_tokens[i]),
                        float(q.cache_hit_ratio[i]), dataset_tag=spec.profile.name) for i in range(q.n)]


def solo_baseline_ttft(spec: RequestSpec, config: ClusterConfig, models: Optional[CostModelPair] = None) -> float:
    """workload.cpp:101-115 (the models do not enter the solo timing)."""
    q, s = _q1(spec)
    out = C.c_double()
    check(lib.tsb_solo_baseline_ttft(C.byref(s), 0, C.byref(config.struct()), C.byref(out)))
    return out.value


def assign_slos_queue(q: QueueArrays, config: ClusterConfig, factors: Sequence[float], seed: int) -> QueueArrays:
    """assign_slos (workload.cpp:117-135) in place on a queue: sets deadline + HAS_DEADLINE."""
    f = np.ascontiguousarray(factors, np.float64)
    out = np.empty(q.n, np.float64)
    check(lib.tsb_assign_slos(q.n, C.byref(q.struct()), C.byref(config.struct()), f.ctypes.data, len(f), int(seed),
                              out.ctypes.data))
    q.deadline[:] = out
    q.flags |= capi.HAS_DEADLINE
    return q


def assign_slos(requests: Sequence[RequestSpec], config: ClusterConfig, models: Optional[CostModelPair],
                factors: Sequence[float], seed: int) -> list[RequestSpec]:
    q = assign_slos_queue(QueueArrays.from_specs(requests), config, factors, seed)
    return [RequestSpec(r.id, r.arrival_time, r.context_tokens, r.query_tokens, r.cache_hit_ratio,
                        float(q.deadline[i]), r.measured_cost, r.dataset_tag) for i, r in enumerate(requests)]


# ---- engine.hpp TierLedger --------------------------------------------------------------------
class TierLedger:
    """engine.hpp:22-53 -- the libtsb byte ledger (tsb_ledger_*), the same object the L1 paged
    allocator (ingest.PagedKVCache) runs its grant/defer decisions through."""

    class Outcome(enum.IntEnum):
        Granted = 0
        Deferred = 1

    Granted, Deferred = Outcome.Granted, Outcome.Deferred

    def __init__(self, tier: Tier, capacity: int):
        h = C.c_void_p()
        check(lib.tsb_ledger_create(int(tier), int(capacity), C.byref(h)))
        self._h = h
        self._tier = Tier(tier)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:
            lib.tsb_ledger_destroy(h)
            self._h = None

    def request(self, request_id: int, block_index: int, nbytes: int) -> "TierLedger.Outcome":
        g = C.c_int()
        check(lib.tsb_ledger_request(self._h, int(request_id), int(block_index), int(nbytes), C.byref(g)))
        return self.Granted if g.value else self.Deferred

    def release(self, nbytes: int) -> list:
        n = C.c_int64()
        cap = max(16, self.deferred_count())
        out = (capi.Grant * cap)()
        check(lib.tsb_ledger_release(self._h, int(nbytes), out, cap, C.byref(n)))
        return [Pending(out[i].request_id, out[i].block_index, out[i].bytes) for i in range(n.value)]

    def tier(self) -> Tier:
        return self._tier

    def capacity(self) -> int:
        return lib.tsb_ledger_capacity(self._h)

    def reserved(self) -> int:
        return lib.tsb_ledger_reserved(self._h)

    def deferred_count(self) -> int:
        return lib.tsb_ledger_deferred(self._h)


@dataclass
class Pending:
    """TierLedger::Pending (engine.hpp:26-30)"""

    request_id: int
    block_index: int
    bytes: int
