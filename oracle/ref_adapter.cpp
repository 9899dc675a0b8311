// ref_adapter.cpp — extern "C" shim over the reference's own sources.
//
// TEST INFRASTRUCTURE ONLY.  Compiled together with /root/reference/proj/core/src/*.cpp
// (in place, never copied) under -Dtiersim=tiersim_ref, so every `tiersim::` below is the
// reference implementation.  Exposes plain-pointer entry points so pytest (ctypes) and the
// golden-vector generator can run the reference on the same inputs as the GPU path.
#include <algorithm>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "tiersim/cost_model.hpp"
#include "tiersim/engine.hpp"
#include "tiersim/error.hpp"
#include "tiersim/scheduler.hpp"
#include "tiersim/types.hpp"
#include "tiersim/workload.hpp"
#include "../oracle/tsb_oracle.h"

namespace {

thread_local std::string g_msg;

int map_exception() {
  try {
    throw;
  } catch (const tiersim::ValidationError& e) {
    g_msg = e.what();
    return ORC_VALIDATION;
  } catch (const tiersim::CapacityError& e) {
    g_msg = e.what();
    return ORC_CAPACITY;
  } catch (const tiersim::MissingDeadline& e) {
    g_msg = e.what();
    return ORC_MISSING_DEADLINE;
  } catch (const tiersim::DegenerateFit& e) {
    g_msg = e.what();
    return ORC_DEGENERATE_FIT;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return 99;
  }
}

tiersim::ClusterConfig to_cfg(const orc_cluster* c) {
  tiersim::ClusterConfig cfg;
  cfg.network_bandwidth = c->network_bandwidth;
  cfg.pcie_bandwidth = c->pcie_bandwidth;
  cfg.transfer_base_latency = c->transfer_base_latency;
  cfg.l1_capacity = c->l1_capacity;
  cfg.l2_capacity = c->l2_capacity;
  cfg.bytes_per_token = c->bytes_per_token;
  cfg.block_size_tokens = c->block_size_tokens;
  cfg.compute_base = c->compute_base;
  cfg.compute_per_token = c->compute_per_token;
  cfg.compute_quadratic = c->compute_quadratic;
  cfg.allocation_mode = c->allocation_mode ? tiersim::AllocationMode::Reactive
                                           : tiersim::AllocationMode::Proactive;
  cfg.control_mode =
      c->control_mode ? tiersim::ControlMode::Decoupled : tiersim::ControlMode::Coupled;
  return cfg;
}

tiersim::RequestSpec to_spec(const orc_queue* q, int64_t i) {
  tiersim::RequestSpec s;
  s.id = q->id[i];
  s.arrival_time = q->arrival[i];
  s.context_tokens = q->context_tokens[i];
  s.query_tokens = q->query_tokens[i];
  s.cache_hit_ratio = q->cache_hit_ratio[i];
  if (q->flags[i] & ORC_HAS_DEADLINE) s.deadline = q->deadline[i];
  if (q->flags[i] & ORC_HAS_MEASURED)
    s.measured_cost = tiersim::MeasuredCost{q->measured_t_load[i], q->measured_t_comp[i]};
  return s;
}

tiersim::CostModelPair to_models(const double m[4]) {
  tiersim::CostModelPair p;
  p.load.slope = m[0];
  p.load.intercept = m[1];
  p.comp.slope = m[2];
  p.comp.intercept = m[3];
  return p;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_msg.c_str(); }

int ref_kv_bytes_per_token(int64_t l, int64_t h, int64_t d, int64_t e, int64_t* out) {
  try {
    *out = tiersim::kv_bytes_per_token(l, h, d, e);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// make_request_state (types.cpp:103-111): cached, compute, plan size and per-block bytes.
int ref_block_plan(const orc_queue* q, int64_t i, const orc_cluster* c, int64_t* cached,
                   int64_t* compute, int64_t* n_blocks, int64_t* block_tokens,
                   int64_t* block_bytes) {
  try {
    const auto cfg = to_cfg(c);
    const auto st = tiersim::make_request_state(to_spec(q, i), cfg);
    *cached = st.cached_tokens;
    *compute = st.compute_tokens;
    *n_blocks = static_cast<int64_t>(st.blocks.size());
    *block_tokens = st.blocks.empty() ? 0 : st.blocks.front().tokens;
    *block_bytes = st.blocks.empty() ? 0 : st.blocks.front().bytes;
    for (std::size_t b = 0; b < st.blocks.size(); ++b) {
      if (st.blocks[b].block_index != static_cast<int32_t>(b) ||
          st.blocks[b].request_id != q->id[i])
        return 98;
    }
    return 0;
  } catch (...) {
    return map_exception();
  }
}

void ref_cost_models_from_config(const orc_cluster* c, double out[4]) {
  const auto m = tiersim::cost_models_from_config(to_cfg(c));
  out[0] = m.load.slope;
  out[1] = m.load.intercept;
  out[2] = m.comp.slope;
  out[3] = m.comp.intercept;
}

int ref_fit_linear(int64_t n, const int64_t* tokens, const double* seconds, double* out4) {
  try {
    std::vector<tiersim::TokenSample> s(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) s[i] = {tokens[i], seconds[i]};
    const auto fit = tiersim::fit_linear(s);
    out4[0] = fit.model.slope;
    out4[1] = fit.model.intercept;
    out4[2] = fit.slope_clamped;
    out4[3] = fit.intercept_clamped;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// estimate_service_cost + priority_key per request, in queue order.
int ref_score_queue(int64_t n, const orc_queue* q, int policy, const double m[4],
                    const orc_cluster* c, double* t_load, double* t_comp, double* primary,
                    int64_t* err_index) {
  *err_index = -1;
  const auto cfg = to_cfg(c);
  const auto models = to_models(m);
  const auto pol = static_cast<tiersim::PolicyKind>(policy);
  for (int64_t i = 0; i < n; ++i) {
    try {
      const auto spec = to_spec(q, i);
      const auto cost = tiersim::estimate_service_cost(spec, models.load, models.comp, cfg);
      const auto key = tiersim::priority_key(spec, pol, cost, 0.0);
      t_load[i] = cost.t_load;
      t_comp[i] = cost.t_comp;
      primary[i] = key.primary;
    } catch (...) {
      *err_index = i;
      return map_exception();
    }
  }
  return 0;
}

// std::sort with PriorityKey::operator< over keys from priority_key.
int ref_sort_order(int64_t n, const orc_queue* q, int policy, const double m[4],
                   const orc_cluster* c, int64_t* order) {
  try {
    const auto cfg = to_cfg(c);
    const auto models = to_models(m);
    const auto pol = static_cast<tiersim::PolicyKind>(policy);
    std::vector<std::pair<tiersim::PriorityKey, int64_t>> keys(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      const auto spec = to_spec(q, i);
      const auto cost = tiersim::estimate_service_cost(spec, models.load, models.comp, cfg);
      keys[i] = {tiersim::priority_key(spec, pol, cost, 0.0), i};
    }
    std::sort(keys.begin(), keys.end(),
              [](const auto& a, const auto& b) { return a.first < b.first; });
    for (int64_t i = 0; i < n; ++i) order[i] = keys[i].second;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// The reference drain: repeated pick_next with a CostMap (scheduler.cpp:93-100,
// test_scheduler.cpp:26-31).  O(n^2).
int ref_drain_order(int64_t n, const orc_queue* q, int policy, const double m[4],
                    const orc_cluster* c, int64_t* order) {
  try {
    const auto cfg = to_cfg(c);
    const auto models = to_models(m);
    const auto pol = static_cast<tiersim::PolicyKind>(policy);
    std::vector<tiersim::RequestSpec> queue;
    tiersim::CostMap costs;
    std::vector<int64_t> index_of;
    for (int64_t i = 0; i < n; ++i) {
      queue.push_back(to_spec(q, i));
      costs[q->id[i]] =
          tiersim::estimate_service_cost(queue.back(), models.load, models.comp, cfg);
    }
    std::unordered_map<int64_t, int64_t> pos;
    for (int64_t i = 0; i < n; ++i) pos[q->id[i]] = i;
    int64_t k = 0;
    while (auto picked = tiersim::pick_next(queue, pol, costs, 0.0)) order[k++] = pos[picked->id];
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// --- TierLedger -------------------------------------------------------------
void* ref_ledger_new(int tier, int64_t capacity) {
  try {
    return new tiersim::TierLedger(static_cast<tiersim::Tier>(tier), capacity);
  } catch (...) {
    map_exception();
    return nullptr;
  }
}
void ref_ledger_free(void* l) { delete static_cast<tiersim::TierLedger*>(l); }
int ref_ledger_request(void* l, int64_t rid, int32_t blk, int64_t bytes, int* granted) {
  try {
    *granted = static_cast<tiersim::TierLedger*>(l)->request(rid, blk, bytes) ==
               tiersim::TierLedger::Outcome::Granted;
    return 0;
  } catch (...) {
    return map_exception();
  }
}
int ref_ledger_release(void* l, int64_t bytes, int64_t* rid, int32_t* blk, int64_t* b,
                       int64_t cap, int64_t* n) {
  try {
    const auto g = static_cast<tiersim::TierLedger*>(l)->release(bytes);
    *n = static_cast<int64_t>(g.size());
    for (int64_t i = 0; i < *n && i < cap; ++i) {
      rid[i] = g[i].request_id;
      blk[i] = g[i].block_index;
      b[i] = g[i].bytes;
    }
    return 0;
  } catch (...) {
    *n = 0;
    return map_exception();
  }
}
int64_t ref_ledger_reserved(void* l) { return static_cast<tiersim::TierLedger*>(l)->reserved(); }
int64_t ref_ledger_deferred(void* l) {
  return static_cast<int64_t>(static_cast<tiersim::TierLedger*>(l)->deferred_count());
}

uint64_t ref_config_fingerprint(const orc_cluster* c, int policy, uint64_t seed) {
  return tiersim::config_fingerprint(to_cfg(c), static_cast<tiersim::PolicyKind>(policy), seed);
}

// generate_workload (workload.cpp:70-99).  profile: builtin name or "custom" with the
// given mean/cv.  Returns the number of requests written (<= cap) or -status.
int64_t ref_generate_workload(const char* profile, double ctx_mean, double ctx_cv,
                              double q_mean, double q_cv, int64_t count, double qps,
                              uint64_t seed, int hit_kind, double hit_fixed,
                              const double* choices, int64_t n_choices, int64_t cap,
                              int64_t* id, double* arrival, int64_t* ctx, int64_t* query,
                              double* hit) {
  try {
    tiersim::WorkloadSpec w;
    if (std::string(profile) == "custom") {
      w.profile = {"custom", count, ctx_mean, ctx_cv, q_mean, q_cv};
    } else {
      w.profile = tiersim::builtin_profile(profile);
    }
    w.qps = qps;
    w.count = count;
    w.seed = seed;
    if (hit_kind == 0)
      w.hit_ratio_source = tiersim::HitRatioSource::fixed(hit_fixed);
    else
      w.hit_ratio_source = tiersim::HitRatioSource::uniform_choice(
          std::vector<double>(choices, choices + n_choices));
    const auto reqs = tiersim::generate_workload(w);
    const int64_t n = static_cast<int64_t>(reqs.size());
    for (int64_t i = 0; i < n && i < cap; ++i) {
      id[i] = reqs[i].id;
      arrival[i] = reqs[i].arrival_time;
      ctx[i] = reqs[i].context_tokens;
      query[i] = reqs[i].query_tokens;
      hit[i] = reqs[i].cache_hit_ratio;
    }
    return n;
  } catch (...) {
    return -map_exception();
  }
}

// assign_slos (workload.cpp:117-135): deadlines for a queue (input order).
int ref_assign_slos(int64_t n, const orc_queue* q, const orc_cluster* c, const double m[4],
                    const double* factors, int64_t n_factors, uint64_t seed, double* deadline) {
  try {
    std::vector<tiersim::RequestSpec> reqs;
    for (int64_t i = 0; i < n; ++i) reqs.push_back(to_spec(q, i));
    const auto out = tiersim::assign_slos(reqs, to_cfg(c), to_models(m),
                                          std::span<const double>(factors, static_cast<size_t>(n_factors)), seed);
    for (int64_t i = 0; i < n; ++i) deadline[i] = *out[static_cast<size_t>(i)].deadline;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// run_simulation (engine.cpp:536-552) for the sim-vs-real comparison: per-request
// (scheduled, l1_resident, first_token, ttft) in input order; returns mean TTFT via out.
int ref_run_simulation(int64_t n, const orc_queue* q, const orc_cluster* c, int policy,
                       const double m[4], uint64_t seed, double* ttft, double* mean_ttft) {
  try {
    std::vector<tiersim::RequestSpec> reqs;
    for (int64_t i = 0; i < n; ++i) reqs.push_back(to_spec(q, i));
    tiersim::RunOptions opts;
    opts.record_trace = false;
    const auto rep = tiersim::run_simulation(reqs, to_cfg(c),
                                             static_cast<tiersim::PolicyKind>(policy),
                                             to_models(m), seed, opts);
    std::unordered_map<int64_t, double> by_id;
    for (const auto& r : rep.records) by_id[r.id] = r.ttft;
    for (int64_t i = 0; i < n; ++i) ttft[i] = by_id[q->id[i]];
    *mean_ttft = rep.mean_ttft;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

}  // extern "C"
