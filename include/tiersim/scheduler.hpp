// tiersim/scheduler.hpp — queue-ordering policies of the reference (core/include/tiersim/scheduler.hpp)
// with the queue-wide operations on the GPU: BatchScorer runs K4 (estimate_service_cost +
// priority_key) and K5 (the order PriorityKey::operator< induces, == the pick_next drain) through
// tsb_score_queue.  best_request_index / pick_next keep their reference signatures on top of it.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "tiersim/cost_model.hpp"
#include "tiersim/types.hpp"

namespace tiersim {

enum class PolicyKind : std::uint8_t { Fifo, SjfPt, SjfCost, Edf, Lstf };

inline std::optional<PolicyKind> policy_from_name(std::string_view n) {
  if (n == "fifo") return PolicyKind::Fifo;
  if (n == "sjf-pt") return PolicyKind::SjfPt;
  if (n == "sjf-cost") return PolicyKind::SjfCost;
  if (n == "edf") return PolicyKind::Edf;
  if (n == "lstf") return PolicyKind::Lstf;
  return std::nullopt;
}

inline std::string_view policy_name(PolicyKind p) {
  switch (p) {
    case PolicyKind::Fifo: return "fifo";
    case PolicyKind::SjfPt: return "sjf-pt";
    case PolicyKind::SjfCost: return "sjf-cost";
    case PolicyKind::Edf: return "edf";
    case PolicyKind::Lstf: return "lstf";
  }
  return "?";
}

inline std::span<const PolicyKind> all_policies() {
  static constexpr std::array<PolicyKind, 5> k = {PolicyKind::Fifo, PolicyKind::SjfPt,
                                                  PolicyKind::SjfCost, PolicyKind::Edf,
                                                  PolicyKind::Lstf};
  return k;
}

struct PriorityKey {
  double primary = 0.0;
  double arrival = 0.0;
  std::int64_t id = 0;
  friend bool operator<(const PriorityKey& a, const PriorityKey& b) {
    if (a.primary != b.primary) return a.primary < b.primary;
    if (a.arrival != b.arrival) return a.arrival < b.arrival;
    return a.id < b.id;
  }
};

inline double prefill_token_estimate(const RequestSpec& spec) {
  detail::SpecView v(spec);
  double out = 0.0;
  check(tsb_priority_key(&v.q, 0, static_cast<int>(PolicyKind::SjfPt), 0.0, 0.0, &out));
  return out;
}

inline PriorityKey priority_key(const RequestSpec& spec, PolicyKind policy, const ServiceCost& cost,
                                double now) {
  (void)now;  // keys ignore `now` (scheduler.cpp:47)
  detail::SpecView v(spec);
  PriorityKey key;
  key.arrival = spec.arrival_time;
  key.id = spec.id;
  check(tsb_priority_key(&v.q, 0, static_cast<int>(policy), cost.t_load, cost.t_comp, &key.primary));
  return key;
}

using CostMap = std::unordered_map<std::int64_t, ServiceCost>;

/// Struct-of-arrays copy of a RequestSpec queue as tsb_queue expects it.
class QueueSoA {
 public:
  /// costs != nullptr: CostMap semantics (scheduler.cpp:82-83) -- each request's cost is the
  /// map entry (zero when missing), passed as a measured override.
  QueueSoA(std::span<const RequestSpec> q, const CostMap* costs) {
    const std::size_t n = q.size();
    id.resize(n); ctx.resize(n); query.resize(n); flags.resize(n);
    arrival.resize(n); hit.resize(n); deadline.resize(n); ml.resize(n); mc.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
      const RequestSpec& s = q[i];
      id[i] = s.id; ctx[i] = s.context_tokens; query[i] = s.query_tokens;
      arrival[i] = s.arrival_time; hit[i] = s.cache_hit_ratio;
      uint8_t f = 0;
      if (s.deadline) { f |= TSB_HAS_DEADLINE; deadline[i] = *s.deadline; }
      std::optional<MeasuredCost> m = s.measured_cost;
      if (costs) {
        const auto it = costs->find(s.id);
        const ServiceCost c = it != costs->end() ? it->second : ServiceCost{};
        m = MeasuredCost{c.t_load, c.t_comp};
      }
      if (m) { f |= TSB_HAS_MEASURED; ml[i] = m->t_load; mc[i] = m->t_comp; }
      flags[i] = f;
    }
    view = tsb_queue{id.data(), arrival.data(), ctx.data(), query.data(), hit.data(),
                     flags.data(), deadline.data(), ml.data(), mc.data()};
  }
  const tsb_queue* get() const { return &view; }
  int64_t size() const { return static_cast<int64_t>(id.size()); }

 private:
  std::vector<int64_t> id, ctx, query;
  std::vector<uint8_t> flags;
  std::vector<double> arrival, hit, deadline, ml, mc;
  tsb_queue view{};
};

/// The batched GPU scorer (K4 + K5).  One per device and host thread.
class BatchScorer {
 public:
  explicit BatchScorer(int device = 0, int64_t capacity = 1 << 17) {
    tsb_scorer* s = nullptr;
    check(tsb_scorer_create(device, capacity, &s));
    s_.reset(s);
  }
  struct Result {
    std::vector<double> t_load, t_comp, primary;
    std::vector<int64_t> order;  ///< order[k] = queue index picked k-th
  };
  Result score(std::span<const RequestSpec> queue, PolicyKind policy, const CostModelPair& models,
               const ClusterConfig& config, const CostMap* costs = nullptr, void* stream = nullptr) {
    QueueSoA q(queue, costs);
    Result r;
    const std::size_t n = queue.size();
    r.t_load.resize(n); r.t_comp.resize(n); r.primary.resize(n); r.order.resize(n);
    double m[4];
    models.c_abi(m);
    const tsb_cluster c = config.c_abi();
    check(tsb_score_queue(s_.get(), stream, q.size(), q.get(), static_cast<int>(policy), m, &c,
                          r.t_load.data(), r.t_comp.data(), r.primary.data(), r.order.data()));
    return r;
  }
  tsb_scorer* handle() { return s_.get(); }

  /// One scorer per (host thread, current device): a rank bound to cuda:k scores on cuda:k.
  static BatchScorer& shared() {
    const int dev = tsb_current_device();
    static thread_local std::unordered_map<int, std::unique_ptr<BatchScorer>> per_dev;
    auto& s = per_dev[dev];
    if (!s) s = std::make_unique<BatchScorer>(dev);
    return *s;
  }

 private:
  struct Del {
    void operator()(tsb_scorer* s) const { tsb_scorer_destroy(s); }
  };
  std::unique_ptr<tsb_scorer, Del> s_;
};

namespace detail {
/// Priority keys the GPU scorer already computed, by request id.  A key depends only on the
/// request's fields, its CostMap entry and the policy (never on `now`, scheduler.cpp:47), so an
/// engine that calls pick_next in its pump loop pays the GPU round trip once per request, not once
/// per pick; each pick is then the reference's O(n) argmin over cached keys.
struct CachedKey {
  double arrival, hit, deadline, t_load, t_comp, primary;
  std::int64_t ctx, query;
  bool has_deadline, has_cost, has_measured;
  PolicyKind policy;
};
inline std::unordered_map<std::int64_t, CachedKey>& key_cache() {
  static thread_local std::unordered_map<std::int64_t, CachedKey> m;
  return m;
}
inline CachedKey key_fields(const RequestSpec& s, PolicyKind policy, const CostMap& costs) {
  CachedKey k{};
  k.arrival = s.arrival_time;
  k.hit = s.cache_hit_ratio;
  k.ctx = s.context_tokens;
  k.query = s.query_tokens;
  k.has_deadline = s.deadline.has_value();
  k.deadline = s.deadline.value_or(0.0);
  const auto it = costs.find(s.id);
  k.has_cost = it != costs.end();
  k.t_load = k.has_cost ? it->second.t_load : 0.0;
  k.t_comp = k.has_cost ? it->second.t_comp : 0.0;
  k.has_measured = s.measured_cost.has_value();
  k.policy = policy;
  return k;
}
inline bool same_fields(const CachedKey& a, const CachedKey& b) {
  return a.arrival == b.arrival && a.hit == b.hit && a.ctx == b.ctx && a.query == b.query &&
         a.has_deadline == b.has_deadline && a.deadline == b.deadline && a.has_cost == b.has_cost &&
         a.t_load == b.t_load && a.t_comp == b.t_comp && a.has_measured == b.has_measured &&
         a.policy == b.policy;
}
}  // namespace detail

/// The pick_next drain of a fixed queue in one GPU pass: ids in pick order.
inline std::vector<std::int64_t> schedule_order(std::span<const RequestSpec> queue, PolicyKind policy,
                                                const CostMap& costs) {
  const auto r = BatchScorer::shared().score(queue, policy, CostModelPair{}, ClusterConfig{}, &costs);
  std::vector<std::int64_t> ids(queue.size());
  for (std::size_t k = 0; k < queue.size(); ++k) ids[k] = queue[static_cast<std::size_t>(r.order[k])].id;
  return ids;
}

/// scheduler.cpp:75-91.  Keys of requests not seen before (or whose fields, cost or policy
/// changed) are computed by the GPU scorer in one batch; the argmin (first minimum wins) runs over
/// the cached keys, as the reference's scan does.
inline std::optional<std::size_t> best_request_index(std::span<const RequestSpec> queue,
                                                     PolicyKind policy, const CostMap& costs,
                                                     double now) {
  (void)now;
  if (queue.empty()) return std::nullopt;
  auto& cache = detail::key_cache();
  if (cache.size() > 4 * queue.size() + 4096) cache.clear();  // bounded: drop finished requests
  std::vector<RequestSpec> fresh;
  std::vector<detail::CachedKey> fresh_fields;
  std::vector<const detail::CachedKey*> keys(queue.size(), nullptr);
  for (std::size_t i = 0; i < queue.size(); ++i) {
    const detail::CachedKey f = detail::key_fields(queue[i], policy, costs);
    const auto it = cache.find(queue[i].id);
    if (it != cache.end() && detail::same_fields(it->second, f)) {
      keys[i] = &it->second;
    } else {
      fresh.push_back(queue[i]);
      fresh_fields.push_back(f);
    }
  }
  if (!fresh.empty()) {
    const auto r = BatchScorer::shared().score(fresh, policy, CostModelPair{}, ClusterConfig{}, &costs);
    for (std::size_t k = 0; k < fresh.size(); ++k) {
      fresh_fields[k].primary = r.primary[k];
      cache[fresh[k].id] = fresh_fields[k];
    }
    for (std::size_t i = 0; i < queue.size(); ++i)
      if (!keys[i]) keys[i] = &cache.at(queue[i].id);
  }
  std::size_t best = 0;
  PriorityKey best_key{keys[0]->primary, queue[0].arrival_time, queue[0].id};
  for (std::size_t i = 1; i < queue.size(); ++i) {
    const PriorityKey k{keys[i]->primary, queue[i].arrival_time, queue[i].id};
    if (k < best_key) {
      best = i;
      best_key = k;
    }
  }
  return best;
}

/// scheduler.cpp:93-100
inline std::optional<RequestSpec> pick_next(std::vector<RequestSpec>& queue, PolicyKind policy,
                                            const CostMap& costs, double now) {
  const auto idx = best_request_index(queue, policy, costs, now);
  if (!idx) return std::nullopt;
  RequestSpec picked = std::move(queue[*idx]);
  queue.erase(queue.begin() + static_cast<std::ptrdiff_t>(*idx));
  return picked;
}

}  // namespace tiersim
