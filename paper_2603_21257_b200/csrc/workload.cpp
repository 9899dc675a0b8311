// workload.cpp — C ABI: the synthetic request stream and SLO assignment the configs[3]/[4]
// queues are drawn from (tsb_generate_workload, tsb_solo_baseline_ttft, tsb_assign_slos).
//
// Restates core/src/workload.cpp:31-36, 70-99, 101-135 and core/include/tiersim/rng.hpp:19-70
// so the product makes its own queues: the same seed gives the same RequestSpecs, bit for bit,
// as the reference's generate_workload (pinned against the compiled reference in
// tests/test_capi_cpu.py).  std::mt19937_64 is fully specified by the C++ standard; the
// inverse-CDF and Box-Muller arithmetic is evaluated in the reference's order with
// -ffp-contract=off.
//
// solo_baseline_ttft (workload.cpp:101-115) runs the reference DES on one request in an empty
// decoupled system.  Alone, that run is a fixed recurrence -- every hop starts at an event time
// of the previous one -- so it is evaluated here in closed form with the same additions:
//   net_end[b]   = net_end[b-1] + (lat + bytes/net_bw)                    (engine.cpp:405-425)
//   pcie_end[b]  = max(net_end[b], pcie_end[b-1]) + (lat + bytes/pcie_bw) (engine.cpp:427-446)
//   first_token  = pcie_end[last] + compute_duration                      (engine.cpp:448-473)
// with the measured-cost pseudo-block of engine.cpp:187-198.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <string>

#include "common.cuh"

using tsb::fail;

namespace {

constexpr uint64_t kHitStreamSalt = 0x9e3779b97f4a7c15ull;  // workload.cpp:18
constexpr uint64_t kSloStreamSalt = 0xd1b54a32d192ed03ull;  // workload.cpp:19
constexpr double kMinArrivalGap = 1e-6;                     // workload.cpp:20

// tiersim::Rng (rng.hpp:19-70).
class Rng {
 public:
  explicit Rng(uint64_t seed) : gen_(seed) {}
  double uniform01() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
  double exponential() { return -std::log(1.0 - uniform01()); }
  double normal() {
    if (has_spare_) {
      has_spare_ = false;
      return spare_;
    }
    const double u1 = 1.0 - uniform01();
    const double u2 = uniform01();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * std::acos(-1.0) * u2;
    spare_ = radius * std::sin(angle);
    has_spare_ = true;
    return radius * std::cos(angle);
  }
  double lognormal_mean_cv(double mean, double cv) {
    if (cv <= 0.0) return mean;
    const double sigma2 = std::log1p(cv * cv);
    const double mu = std::log(mean) - 0.5 * sigma2;
    return std::exp(mu + std::sqrt(sigma2) * normal());
  }
  double choice(const double* v, int64_t n) {
    const auto idx = static_cast<size_t>(uniform01() * static_cast<double>(n));
    return v[idx < static_cast<size_t>(n) ? idx : static_cast<size_t>(n) - 1];
  }

 private:
  std::mt19937_64 gen_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

int64_t sample_tokens(Rng& rng, double mean, double cv) {  // workload.cpp:63-66
  return std::max<int64_t>(1, std::llround(rng.lognormal_mean_cv(mean, cv)));
}

}  // namespace

extern "C" {

tsb_status tsb_builtin_profile(const char* name, tsb_workload_spec* out) {
  // builtin_profile (workload.cpp:31-36)
  const std::string n = name ? name : "";
  if (n == "loogle") *out = {120, 28100.0, 0.5, 28.0, 0.5, 1.0, 0, 0, 1.0, nullptr, 0, 0};
  else if (n == "icl") *out = {120, 28300.0, 0.5, 61.0, 0.5, 1.0, 0, 0, 1.0, nullptr, 0, 0};
  else if (n == "code") *out = {100, 38300.0, 0.5, 209.0, 0.5, 1.0, 0, 0, 1.0, nullptr, 0, 0};
  else return fail(TSB_UNKNOWN_PROFILE, "unknown dataset profile: " + n);
  return TSB_OK;
}

tsb_status tsb_workload_validate(const tsb_workload_spec* w) {
  // DatasetProfile::validate, HitRatioSource::validate, WorkloadSpec::validate (workload.cpp:23-61)
  if (w->num_requests < 1) return fail(TSB_VALIDATION, "profile: num_requests must be >= 1");
  if (!(w->context_tokens_mean > 0.0) || !(w->query_tokens_mean > 0.0))
    return fail(TSB_VALIDATION, "profile: token means must be > 0");
  if (w->context_tokens_cv < 0.0 || w->query_tokens_cv < 0.0)
    return fail(TSB_VALIDATION, "profile: token cv must be >= 0");
  if (w->hit_kind == 0) {
    if (!(w->hit_fixed >= 0.0 && w->hit_fixed <= 1.0))
      return fail(TSB_VALIDATION, "hit_ratio_source: fixed value must be in [0, 1]");
  } else {
    if (w->n_hit_choices < 1 || !w->hit_choices)
      return fail(TSB_VALIDATION, "hit_ratio_source: uniform set must be non-empty");
    for (int64_t k = 0; k < w->n_hit_choices; ++k)
      if (!(w->hit_choices[k] >= 0.0 && w->hit_choices[k] <= 1.0))
        return fail(TSB_VALIDATION, "hit_ratio_source: choices must be in [0, 1]");
  }
  if (!(w->qps > 0.0)) return fail(TSB_VALIDATION, "workload: qps must be > 0");
  return TSB_OK;
}

int64_t tsb_workload_count(const tsb_workload_spec* w) {
  return w->count > 0 ? w->count : w->num_requests;  // WorkloadSpec::effective_count
}

tsb_status tsb_generate_workload(const tsb_workload_spec* w, int64_t cap, int64_t* id,
                                 double* arrival, int64_t* context_tokens,
                                 int64_t* query_tokens, double* cache_hit_ratio, int64_t* n_out) {
  TSB_TRY(tsb_workload_validate(w));
  const int64_t count = tsb_workload_count(w);
  if (cap < count)
    return fail(TSB_VALIDATION, "generate_workload: output capacity " + std::to_string(cap) +
                                    " < " + std::to_string(count) + " requests");
  Rng rng(w->seed);
  Rng hit_rng(w->seed ^ kHitStreamSalt);
  double clock = 0.0;
  for (int64_t i = 0; i < count; ++i) {
    id[i] = i + 1;
    clock += std::max(rng.exponential() / w->qps, kMinArrivalGap);
    arrival[i] = clock;
    context_tokens[i] = sample_tokens(rng, w->context_tokens_mean, w->context_tokens_cv);
    query_tokens[i] = sample_tokens(rng, w->query_tokens_mean, w->query_tokens_cv);
    cache_hit_ratio[i] = w->hit_kind == 0 ? w->hit_fixed : hit_rng.choice(w->hit_choices, w->n_hit_choices);
  }
  *n_out = count;
  return TSB_OK;
}

tsb_status tsb_solo_baseline_ttft(const tsb_queue* q, int64_t i, const tsb_cluster* c,
                                  double* ttft) {
  TSB_TRY(tsb_cluster_validate(c));
  int64_t cached = 0, compute = 0, nb = 0, bt = 0, bb = 0;
  TSB_TRY(tsb_derive_block_plan(q, i, c, &cached, &compute, &nb, &bt, &bb));
  const bool measured = q->flags && (q->flags[i] & TSB_HAS_MEASURED);
  double net = 0.0, pcie = 0.0, comp = 0.0;
  int64_t blocks = nb, total_bytes = nb * bb;
  if (measured) {  // engine.cpp:187-198: one pseudo-block whose net hop is t_load
    blocks = q->measured_t_load[i] > 0.0 ? 1 : 0;
    total_bytes = blocks ? std::max<int64_t>(cached, 1) * c->bytes_per_token : 0;
    net = q->measured_t_load[i];
    comp = q->measured_t_comp[i];
  } else {
    net = c->transfer_base_latency + static_cast<double>(bb) / c->network_bandwidth;
    pcie = c->transfer_base_latency + static_cast<double>(bb) / c->pcie_bandwidth;
    const auto ct = static_cast<double>(compute);
    comp = c->compute_base + c->compute_per_token * ct + c->compute_quadratic * ct * ct;
  }
  if (total_bytes > c->l1_capacity || total_bytes > c->l2_capacity)  // engine.cpp:213-217
    return fail(TSB_CAPACITY, "request " + std::to_string(q->id[i]) + ": " +
                                  std::to_string(total_bytes) + " resident bytes can never fit");
  double net_end = 0.0, pcie_end = 0.0;
  for (int64_t b = 0; b < blocks; ++b) {
    net_end = net_end + net;
    pcie_end = std::max(net_end, pcie_end) + pcie;
  }
  const double first_token = pcie_end + comp;
  *ttft = first_token - 0.0;  // solo.arrival_time = 0 (workload.cpp:104), metrics.cpp:97
  return TSB_OK;
}

tsb_status tsb_assign_slos(int64_t n, const tsb_queue* q, const tsb_cluster* c,
                           const double* factors, int64_t n_factors, uint64_t seed,
                           double* deadline_out) {
  // assign_slos (workload.cpp:117-135).  The solo run uses decoupled control (:107); the
  // closed form above does not depend on the control mode or the allocation mode.
  if (n_factors < 1 || !factors) return fail(TSB_VALIDATION, "assign_slos: factor set must be non-empty");
  for (int64_t k = 0; k < n_factors; ++k)
    if (!(factors[k] > 1.0)) return fail(TSB_VALIDATION, "assign_slos: factors must be > 1");
  Rng rng(seed ^ kSloStreamSalt);
  for (int64_t i = 0; i < n; ++i) {
    double base = 0.0;
    TSB_TRY(tsb_solo_baseline_ttft(q, i, c, &base));
    const double f = rng.choice(factors, n_factors);
    deadline_out[i] = q->arrival[i] + f * base;
  }
  return TSB_OK;
}

}  // extern "C"
