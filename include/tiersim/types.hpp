// tiersim/types.hpp — the reference's request / cluster / block types (core/include/tiersim/types.hpp)
// with the planning arithmetic computed by libtsb (tsb_derive_block_plan & co., bit-identical to
// types.cpp:40-118).  Header-only over include/tsb_capi.h.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "tiersim/error.hpp"
#include "tsb_capi.h"

namespace tiersim {

enum class Tier : std::uint8_t { L3, L2, L1 };

inline const char* tier_name(Tier tier) {
  switch (tier) {
    case Tier::L3: return "l3";
    case Tier::L2: return "l2";
    case Tier::L1: return "l1";
  }
  return "?";
}

class TierSet {
 public:
  bool contains(Tier t) const noexcept { return (mask_ & bit(t)) != 0; }
  void insert(Tier t) noexcept { mask_ |= bit(t); }
  void erase(Tier t) noexcept { mask_ &= static_cast<std::uint8_t>(~bit(t)); }
  bool empty() const noexcept { return mask_ == 0; }
  bool operator==(const TierSet&) const = default;

 private:
  static std::uint8_t bit(Tier t) noexcept {
    return static_cast<std::uint8_t>(1u << static_cast<unsigned>(t));
  }
  std::uint8_t mask_ = 0;
};

struct MeasuredCost {
  double t_load = 0.0;
  double t_comp = 0.0;
};

struct RequestSpec;
namespace detail {
/// One RequestSpec viewed as a single-entry tsb_queue (struct-of-arrays of length 1).
struct SpecView {
  int64_t id, ctx, query;
  double arrival, hit, deadline = 0.0, ml = 0.0, mc = 0.0;
  uint8_t flags = 0;
  tsb_queue q{};
  explicit SpecView(const RequestSpec& s);
  SpecView(const SpecView&) = delete;
};
}  // namespace detail

struct RequestSpec {
  std::int64_t id = 0;
  double arrival_time = 0.0;
  std::int64_t context_tokens = 0;
  std::int64_t query_tokens = 1;
  double cache_hit_ratio = 1.0;
  std::optional<double> deadline;
  std::optional<MeasuredCost> measured_cost;
  std::string dataset_tag;

  void validate() const {  // types.cpp:40-54
    detail::SpecView v(*this);
    check(tsb_request_validate(&v.q, 0));
  }
};

namespace detail {
inline SpecView::SpecView(const RequestSpec& s)
    : id(s.id), ctx(s.context_tokens), query(s.query_tokens), arrival(s.arrival_time),
      hit(s.cache_hit_ratio) {
  if (s.deadline) {
    deadline = *s.deadline;
    flags |= TSB_HAS_DEADLINE;
  }
  if (s.measured_cost) {
    ml = s.measured_cost->t_load;
    mc = s.measured_cost->t_comp;
    flags |= TSB_HAS_MEASURED;
  }
  q = tsb_queue{&id, &arrival, &ctx, &query, &hit, &flags, &deadline, &ml, &mc};
}
}  // namespace detail

enum class AllocationMode : std::uint8_t { Proactive, Reactive };
enum class ControlMode : std::uint8_t { Coupled, Decoupled };

inline const char* allocation_mode_name(AllocationMode m) {
  return m == AllocationMode::Proactive ? "proactive" : "reactive";
}
inline const char* control_mode_name(ControlMode m) {
  return m == ControlMode::Coupled ? "coupled" : "decoupled";
}
inline std::optional<AllocationMode> allocation_mode_from_name(const std::string& n) {
  if (n == "proactive") return AllocationMode::Proactive;
  if (n == "reactive") return AllocationMode::Reactive;
  return std::nullopt;
}
inline std::optional<ControlMode> control_mode_from_name(const std::string& n) {
  if (n == "coupled") return ControlMode::Coupled;
  if (n == "decoupled") return ControlMode::Decoupled;
  return std::nullopt;
}

struct ClusterConfig {
  double network_bandwidth = 50e9;
  double pcie_bandwidth = 64e9;
  double transfer_base_latency = 10e-6;
  std::int64_t l1_capacity = 80'000'000'000;
  std::int64_t l2_capacity = 128'000'000'000;
  std::int64_t bytes_per_token = 131072;
  std::int64_t block_size_tokens = 256;
  double compute_base = 2e-3;
  double compute_per_token = 4e-5;
  double compute_quadratic = 0.0;
  AllocationMode allocation_mode = AllocationMode::Proactive;
  ControlMode control_mode = ControlMode::Decoupled;

  tsb_cluster c_abi() const {
    return tsb_cluster{network_bandwidth, pcie_bandwidth,   transfer_base_latency,
                       l1_capacity,       l2_capacity,      bytes_per_token,
                       block_size_tokens, compute_base,     compute_per_token,
                       compute_quadratic, static_cast<int32_t>(allocation_mode),
                       static_cast<int32_t>(control_mode)};
  }
  void validate() const {  // types.cpp:56-71
    const tsb_cluster c = c_abi();
    check(tsb_cluster_validate(&c));
  }
};

struct KVBlock {
  std::int64_t request_id = 0;
  std::int32_t block_index = 0;
  std::int64_t tokens = 0;
  std::int64_t bytes = 0;
  Tier residency = Tier::L3;
  TierSet allocated_at;
};

struct Timestamps {
  double arrival = 0.0;
  std::optional<double> scheduled;
  std::optional<double> net_first_dispatch;
  std::optional<double> l2_resident;
  std::optional<double> l1_resident;
  std::optional<double> compute_start;
  std::optional<double> first_token;
};

struct RequestState {
  RequestSpec spec;
  std::int64_t cached_tokens = 0;
  std::int64_t compute_tokens = 0;
  std::vector<KVBlock> blocks;
  Timestamps ts;
};

namespace detail {
struct Plan {
  int64_t cached = 0, compute = 0, n = 0, tokens = 0, bytes = 0;
};
inline Plan plan_of(const RequestSpec& spec, const ClusterConfig& config) {
  detail::SpecView v(spec);
  const tsb_cluster c = config.c_abi();
  Plan p;
  check(tsb_derive_block_plan(&v.q, 0, &c, &p.cached, &p.compute, &p.n, &p.tokens, &p.bytes));
  return p;
}
}  // namespace detail

/// types.cpp:73-79 (floor rule; this form does not validate, like the reference).
inline std::int64_t cached_token_count(const RequestSpec& spec, const ClusterConfig& config) {
  RequestSpec s = spec;
  s.deadline.reset();
  s.measured_cost.reset();
  if (s.query_tokens < 1) s.query_tokens = 1;
  return detail::plan_of(s, config).cached;
}

inline std::int64_t compute_token_count(const RequestSpec& spec, const ClusterConfig& config) {
  return spec.context_tokens + spec.query_tokens - cached_token_count(spec, config);
}

/// types.cpp:85-101 (validates the spec).
inline std::vector<KVBlock> derive_block_plan(const RequestSpec& spec, const ClusterConfig& config) {
  const auto p = detail::plan_of(spec, config);
  std::vector<KVBlock> plan(static_cast<std::size_t>(p.n));
  for (int64_t i = 0; i < p.n; ++i) {
    plan[i].request_id = spec.id;
    plan[i].block_index = static_cast<std::int32_t>(i);
    plan[i].tokens = p.tokens;
    plan[i].bytes = p.bytes;
  }
  return plan;
}

inline RequestState make_request_state(const RequestSpec& spec, const ClusterConfig& config) {
  RequestState st;
  st.spec = spec;
  st.cached_tokens = cached_token_count(spec, config);
  st.compute_tokens = compute_token_count(spec, config);
  st.blocks = derive_block_plan(spec, config);
  st.ts.arrival = spec.arrival_time;
  return st;
}

inline std::int64_t kv_bytes_per_token(std::int64_t layers, std::int64_t kv_heads,
                                       std::int64_t head_dim, std::int64_t dtype_bytes) {
  int64_t out = 0;
  check(tsb_kv_bytes_per_token(layers, kv_heads, head_dim, dtype_bytes, &out));
  return out;
}

}  // namespace tiersim
