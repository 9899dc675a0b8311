// tiersim/workload.hpp — the reference's synthetic request stream (core/include/tiersim/workload.hpp)
// over libtsb: generate_workload, solo_baseline_ttft and assign_slos compute the same streams and
// deadlines as workload.cpp:31-135 (bit-identical; pinned in tests/test_workload_cpu.py).  The
// JSONL import/export of workload.cpp:137-190 is outside the ingest path and not kept.
#pragma once

#include <cstdint>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "tiersim/cost_model.hpp"
#include "tiersim/types.hpp"

namespace tiersim {

struct DatasetProfile {  // workload.hpp:19-28
  std::string name;
  std::int64_t num_requests = 0;
  double context_tokens_mean = 0.0;
  double context_tokens_cv = 0.5;
  double query_tokens_mean = 0.0;
  double query_tokens_cv = 0.5;
};

inline DatasetProfile builtin_profile(std::string_view name) {  // workload.cpp:31-36
  tsb_workload_spec w{};
  check(tsb_builtin_profile(std::string(name).c_str(), &w));
  return {std::string(name), w.num_requests, w.context_tokens_mean, w.context_tokens_cv, w.query_tokens_mean,
          w.query_tokens_cv};
}

struct HitRatioSource {  // workload.hpp:33-45
  enum class Kind : std::uint8_t { Fixed, UniformChoice };
  Kind kind = Kind::Fixed;
  double fixed_value = 1.0;
  std::vector<double> choices;
  static HitRatioSource fixed(double value) { return {Kind::Fixed, value, {}}; }
  static HitRatioSource uniform_choice(std::vector<double> values) {
    return {Kind::UniformChoice, 0.0, std::move(values)};
  }
};

struct WorkloadSpec {  // workload.hpp:55-68
  DatasetProfile profile;
  double qps = 1.0;
  std::int64_t count = 0;
  HitRatioSource hit_ratio_source = HitRatioSource::fixed(1.0);
  std::vector<double> slo_factors;
  std::uint64_t seed = 0;
  std::int64_t effective_count() const { return count > 0 ? count : profile.num_requests; }

  tsb_workload_spec c_abi() const {
    tsb_workload_spec w{};
    w.num_requests = profile.num_requests;
    w.context_tokens_mean = profile.context_tokens_mean;
    w.context_tokens_cv = profile.context_tokens_cv;
    w.query_tokens_mean = profile.query_tokens_mean;
    w.query_tokens_cv = profile.query_tokens_cv;
    w.qps = qps;
    w.count = count;
    w.hit_kind = hit_ratio_source.kind == HitRatioSource::Kind::Fixed ? 0 : 1;
    w.hit_fixed = hit_ratio_source.fixed_value;
    w.hit_choices = hit_ratio_source.choices.data();
    w.n_hit_choices = static_cast<std::int64_t>(hit_ratio_source.choices.size());
    w.seed = seed;
    return w;
  }
  void validate() const {
    const tsb_workload_spec w = c_abi();
    check(tsb_workload_validate(&w));
    for (const double f : slo_factors)
      if (!(f > 1.0)) throw ValidationError("workload: slo factors must be > 1");
  }
};

/// workload.cpp:70-99
inline std::vector<RequestSpec> generate_workload(const WorkloadSpec& spec) {
  spec.validate();
  const tsb_workload_spec w = spec.c_abi();
  const std::int64_t n = tsb_workload_count(&w);
  std::vector<std::int64_t> id(n), ctx(n), query(n);
  std::vector<double> arrival(n), hit(n);
  std::int64_t got = 0;
  check(tsb_generate_workload(&w, n, id.data(), arrival.data(), ctx.data(), query.data(), hit.data(), &got));
  std::vector<RequestSpec> out(static_cast<std::size_t>(got));
  for (std::int64_t i = 0; i < got; ++i) {
    RequestSpec& r = out[static_cast<std::size_t>(i)];
    r.id = id[i];
    r.arrival_time = arrival[i];
    r.context_tokens = ctx[i];
    r.query_tokens = query[i];
    r.cache_hit_ratio = hit[i];
    r.dataset_tag = spec.profile.name;
  }
  return out;
}

/// workload.cpp:101-115 (the models do not enter the solo timing)
inline double solo_baseline_ttft(const RequestSpec& spec, const ClusterConfig& config,
                                 const CostModelPair& /*models*/ = {}) {
  detail::SpecView v(spec);
  const tsb_cluster c = config.c_abi();
  double t = 0.0;
  check(tsb_solo_baseline_ttft(&v.q, 0, &c, &t));
  return t;
}

/// workload.cpp:117-135
inline std::vector<RequestSpec> assign_slos(std::vector<RequestSpec> requests, const ClusterConfig& config,
                                            const CostModelPair& /*models*/, std::span<const double> factors,
                                            std::uint64_t seed) {
  const tsb_cluster c = config.c_abi();
  // one request at a time through the scalar C ABI, same stream of factor draws as the batch form
  std::vector<std::int64_t> id, ctx, query;
  std::vector<double> arrival, hit, dl, ml, mc, out(requests.size());
  std::vector<std::uint8_t> flags;
  for (const auto& r : requests) {
    id.push_back(r.id);
    ctx.push_back(r.context_tokens);
    query.push_back(r.query_tokens);
    arrival.push_back(r.arrival_time);
    hit.push_back(r.cache_hit_ratio);
    dl.push_back(0.0);
    const bool m = r.measured_cost.has_value();
    ml.push_back(m ? r.measured_cost->t_load : 0.0);
    mc.push_back(m ? r.measured_cost->t_comp : 0.0);
    flags.push_back(m ? TSB_HAS_MEASURED : 0);
  }
  const tsb_queue q{id.data(), arrival.data(), ctx.data(), query.data(), hit.data(),
                    flags.data(), dl.data(), ml.data(), mc.data()};
  check(tsb_assign_slos(static_cast<std::int64_t>(requests.size()), &q, &c, factors.data(),
                        static_cast<std::int64_t>(factors.size()), seed, out.data()));
  for (std::size_t i = 0; i < requests.size(); ++i) requests[i].deadline = out[i];
  return requests;
}

}  // namespace tiersim
