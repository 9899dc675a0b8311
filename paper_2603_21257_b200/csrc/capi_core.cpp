// capi_core.cpp — C ABI: status plumbing, planning arithmetic, cost model, batched scorer
// (K4/K5) and prefix hasher (K3) entry points.
//
// Host arithmetic is compiled with -ffp-contract=off and evaluated in the reference's order,
// so the planning/cost helpers return bit-identical values to the reference functions they
// cite.  Everything data-parallel runs on the device; there is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "hostcopy.h"
#include "kernels.h"

namespace tsb {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

tsb_status fail(tsb_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

tsb_status cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
                 ") in " + what;
  return TSB_CUDA;
}

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

}  // namespace tsb

using tsb::fail;

extern "C" {

const char* tsb_last_error(void) { return tsb::g_last_error.c_str(); }
const char* tsb_version(void) { return "tsb 0.1.0 sm_100a"; }
uint64_t tsb_kernel_launch_count(void) { return tsb::g_launches.load(); }
int tsb_current_device(void) {
  int d = 0;
  return cudaGetDevice(&d) == cudaSuccess ? d : 0;
}

// ---------------------------------------------------------------------------------------
// ClusterConfig (types.hpp:82-97, validate types.cpp:56-71)
// ---------------------------------------------------------------------------------------
void tsb_cluster_default(tsb_cluster* c) {
  c->network_bandwidth = 50e9;
  c->pcie_bandwidth = 64e9;
  c->transfer_base_latency = 10e-6;
  c->l1_capacity = 80'000'000'000;
  c->l2_capacity = 128'000'000'000;
  c->bytes_per_token = 131072;
  c->block_size_tokens = 256;
  c->compute_base = 2e-3;
  c->compute_per_token = 4e-5;
  c->compute_quadratic = 0.0;
  c->allocation_mode = 0;
  c->control_mode = 1;
}

tsb_status tsb_cluster_validate(const tsb_cluster* c) {
  if (!(c->network_bandwidth > 0.0))
    return fail(TSB_VALIDATION, "cluster: network_bandwidth must be > 0");
  if (!(c->pcie_bandwidth > 0.0)) return fail(TSB_VALIDATION, "cluster: pcie_bandwidth must be > 0");
  if (c->transfer_base_latency < 0.0)
    return fail(TSB_VALIDATION, "cluster: transfer_base_latency must be >= 0");
  if (c->l1_capacity <= 0 || c->l2_capacity <= 0)
    return fail(TSB_VALIDATION, "cluster: tier capacities must be > 0");
  if (c->bytes_per_token <= 0) return fail(TSB_VALIDATION, "cluster: bytes_per_token must be > 0");
  if (c->block_size_tokens < 1)
    return fail(TSB_VALIDATION, "cluster: block_size_tokens must be >= 1");
  if (c->compute_base < 0.0 || c->compute_per_token < 0.0 || c->compute_quadratic < 0.0)
    return fail(TSB_VALIDATION, "cluster: compute coefficients must be >= 0");
  return TSB_OK;
}

// config_fingerprint (engine.cpp:500-534): byte-wise FNV-1a over the fields in declaration
// order, each hashed as its in-memory bytes; the three enums are one byte (std::uint8_t).
}  // extern "C"
namespace {
uint64_t fnv1a_bytes(uint64_t h, const void* data, size_t len) {
  const auto* b = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < len; ++i) {
    h ^= b[i];
    h *= tsb::kFnvPrime;
  }
  return h;
}
template <typename T>
uint64_t fnv1a_value(uint64_t h, const T& v) {
  return fnv1a_bytes(h, &v, sizeof(v));
}
}  // namespace
extern "C" {

uint64_t tsb_config_fingerprint(const tsb_cluster* c, int policy, uint64_t seed) {
  uint64_t h = tsb::kFnvOffset;
  h = fnv1a_value(h, c->network_bandwidth);
  h = fnv1a_value(h, c->pcie_bandwidth);
  h = fnv1a_value(h, c->transfer_base_latency);
  h = fnv1a_value(h, c->l1_capacity);
  h = fnv1a_value(h, c->l2_capacity);
  h = fnv1a_value(h, c->bytes_per_token);
  h = fnv1a_value(h, c->block_size_tokens);
  h = fnv1a_value(h, c->compute_base);
  h = fnv1a_value(h, c->compute_per_token);
  h = fnv1a_value(h, c->compute_quadratic);
  h = fnv1a_value(h, static_cast<uint8_t>(c->allocation_mode));
  h = fnv1a_value(h, static_cast<uint8_t>(c->control_mode));
  h = fnv1a_value(h, static_cast<uint8_t>(policy));
  h = fnv1a_value(h, seed);
  return h;
}

// ---------------------------------------------------------------------------------------
// Geometry and plan (types.cpp:73-118)
// ---------------------------------------------------------------------------------------
tsb_status tsb_kv_bytes_per_token(int64_t layers, int64_t kv_heads, int64_t head_dim,
                                  int64_t dtype_bytes, int64_t* out) {
  if (layers < 1 || kv_heads < 1 || head_dim < 1 || dtype_bytes < 1)
    return fail(TSB_VALIDATION, "kv_bytes_per_token: all arguments must be >= 1");
  *out = 2 * layers * kv_heads * head_dim * dtype_bytes;
  return TSB_OK;
}

tsb_status tsb_kv_shape_info(const tsb_kv_shape* s, int64_t* chunk_bytes,
                             int64_t* local_page_bytes, int64_t* local_chunk_bytes) {
  int64_t bpt = 0;
  TSB_TRY(tsb_kv_bytes_per_token(s->layers, s->kv_heads, s->head_dim, s->dtype_bytes, &bpt));
  if (s->chunk_tokens < 1 || s->page_tokens < 1 || s->chunk_tokens % s->page_tokens != 0)
    return fail(TSB_VALIDATION, "kv_shape: chunk_tokens must be a positive multiple of page_tokens");
  if (s->tp_size < 1 || s->kv_heads % s->tp_size != 0 || s->tp_rank < 0 ||
      s->tp_rank >= s->tp_size)
    return fail(TSB_VALIDATION, "kv_shape: tp_size must divide kv_heads and 0 <= tp_rank < tp_size");
  const int64_t run = (s->kv_heads / s->tp_size) * s->head_dim * s->dtype_bytes;
  if (run % 16 != 0)
    return fail(TSB_UNSUPPORTED, "kv_shape: per-rank head slice must be a multiple of 16 bytes");
  if (chunk_bytes) *chunk_bytes = bpt * s->chunk_tokens;
  if (local_page_bytes) *local_page_bytes = bpt / s->tp_size * s->page_tokens;
  if (local_chunk_bytes) *local_chunk_bytes = bpt / s->tp_size * s->chunk_tokens;
  return TSB_OK;
}

// RequestSpec::validate (types.cpp:40-54)
tsb_status tsb_request_validate(const tsb_queue* q, int64_t i) {
  const std::string where = "request " + std::to_string(q->id[i]);
  if (q->context_tokens[i] < 0)
    return fail(TSB_VALIDATION, where + ": context_tokens must be >= 0");
  if (q->query_tokens[i] < 1) return fail(TSB_VALIDATION, where + ": query_tokens must be >= 1");
  const double hit = q->cache_hit_ratio[i];
  if (!(hit >= 0.0 && hit <= 1.0))
    return fail(TSB_VALIDATION, where + ": cache_hit_ratio must be in [0, 1]");
  const uint8_t fl = q->flags ? q->flags[i] : 0;
  if ((fl & TSB_HAS_DEADLINE) && !(q->deadline[i] > q->arrival[i]))
    return fail(TSB_VALIDATION, where + ": deadline must be greater than arrival_time");
  if ((fl & TSB_HAS_MEASURED) && (q->measured_t_load[i] < 0.0 || q->measured_t_comp[i] < 0.0))
    return fail(TSB_VALIDATION, where + ": measured_cost components must be >= 0");
  if (!std::isfinite(q->arrival[i]))
    return fail(TSB_VALIDATION, where + ": arrival_time must be finite");
  return TSB_OK;
}

static int64_t cached_tokens_of(int64_t ctx, double hit, int64_t block) {
  const double hit_tokens = static_cast<double>(ctx) * hit;  // types.cpp:74-75
  const auto blocks =
      static_cast<int64_t>(std::floor(hit_tokens / static_cast<double>(block)));
  return blocks * block;
}

tsb_status tsb_derive_block_plan(const tsb_queue* q, int64_t i, const tsb_cluster* c,
                                 int64_t* cached_tokens, int64_t* compute_tokens,
                                 int64_t* n_blocks, int64_t* block_tokens,
                                 int64_t* block_bytes) {
  TSB_TRY(tsb_request_validate(q, i));  // derive_block_plan validates (types.cpp:86)
  const int64_t cached = cached_tokens_of(q->context_tokens[i], q->cache_hit_ratio[i],
                                          c->block_size_tokens);
  *cached_tokens = cached;
  *compute_tokens = q->context_tokens[i] + q->query_tokens[i] - cached;
  *n_blocks = cached / c->block_size_tokens;
  *block_tokens = cached ? c->block_size_tokens : 0;
  *block_bytes = cached ? c->block_size_tokens * c->bytes_per_token : 0;
  return TSB_OK;
}

// ---------------------------------------------------------------------------------------
// Cost model (cost_model.cpp:14-85)
// ---------------------------------------------------------------------------------------
void tsb_cost_models_from_config(const tsb_cluster* c, double m[4]) {
  const auto bpt = static_cast<double>(c->bytes_per_token);
  m[0] = bpt * (1.0 / c->network_bandwidth + 1.0 / c->pcie_bandwidth) +
         2.0 * c->transfer_base_latency / static_cast<double>(c->block_size_tokens);
  m[1] = 0.0;
  m[2] = c->compute_per_token;
  m[3] = c->compute_base;
}

double tsb_predict(double slope, double intercept, int64_t tokens) {
  return intercept + slope * static_cast<double>(tokens);
}

tsb_status tsb_fit_linear(int64_t n, const int64_t* tokens, const double* seconds, double* slope,
                          double* intercept, int* slope_clamped, int* intercept_clamped) {
  if (n < 2) return fail(TSB_DEGENERATE_FIT, "fit_linear: need at least two samples");
  double mx = 0.0, my = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    mx += static_cast<double>(tokens[i]);
    my += seconds[i];
  }
  const auto dn = static_cast<double>(n);
  mx /= dn;
  my /= dn;
  double sxx = 0.0, sxy = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double dx = static_cast<double>(tokens[i]) - mx;
    sxx += dx * dx;
    sxy += dx * (seconds[i] - my);
  }
  if (sxx == 0.0) return fail(TSB_DEGENERATE_FIT, "fit_linear: all token counts are equal");
  double s = sxy / sxx;
  double b = my - s * mx;
  *slope_clamped = *intercept_clamped = 0;
  if (s < 0.0) {
    s = 0.0;
    *slope_clamped = 1;
  }
  if (b < 0.0) {
    b = 0.0;
    *intercept_clamped = 1;
  }
  *slope = s;
  *intercept = b;
  return TSB_OK;
}

tsb_status tsb_estimate_service_cost(const tsb_queue* q, int64_t i, const double m[4],
                                     const tsb_cluster* c, double* t_load, double* t_comp) {
  const uint8_t fl = q->flags ? q->flags[i] : 0;
  if (fl & TSB_HAS_MEASURED) {  // cost_model.cpp:58-59
    *t_load = q->measured_t_load[i];
    *t_comp = q->measured_t_comp[i];
    return TSB_OK;
  }
  const int64_t cached = cached_tokens_of(q->context_tokens[i], q->cache_hit_ratio[i],
                                          c->block_size_tokens);
  *t_load = cached > 0 ? tsb_predict(m[0], m[1], cached) : 0.0;
  const int64_t ct = q->context_tokens[i] + q->query_tokens[i] - cached;
  double tc = tsb_predict(m[2], m[3], ct);
  if (c->compute_quadratic > 0.0) {
    const auto d = static_cast<double>(ct);
    tc += c->compute_quadratic * d * d;
  }
  *t_comp = tc;
  return TSB_OK;
}

tsb_status tsb_priority_key(const tsb_queue* q, int64_t i, int policy, double t_load,
                            double t_comp, double* primary) {
  const uint8_t fl = q->flags ? q->flags[i] : 0;
  switch (policy) {
    case TSB_FIFO: *primary = q->arrival[i]; return TSB_OK;
    case TSB_SJF_PT: {  // scheduler.cpp:39-43
      const double hit_tokens =
          std::floor(static_cast<double>(q->context_tokens[i]) * q->cache_hit_ratio[i]);
      *primary = static_cast<double>(q->context_tokens[i] + q->query_tokens[i]) - hit_tokens;
      return TSB_OK;
    }
    case TSB_SJF_COST: *primary = t_load + t_comp; return TSB_OK;
    case TSB_EDF:
    case TSB_LSTF:
      if (!(fl & TSB_HAS_DEADLINE))
        return fail(TSB_MISSING_DEADLINE, std::string(policy == TSB_EDF ? "edf" : "lstf") +
                                              ": request " + std::to_string(q->id[i]) +
                                              " has no deadline");
      *primary = policy == TSB_EDF ? q->deadline[i] : q->deadline[i] - (t_load + t_comp);
      return TSB_OK;
    default: return fail(TSB_VALIDATION, "unknown policy");
  }
}

}  // extern "C"

// ---------------------------------------------------------------------------------------
// Scorer object: device scratch for K4 keys and K5 ping-pong buffers.
// ---------------------------------------------------------------------------------------
struct tsb_scorer {
  int device = 0;
  int64_t capacity = 0;
  uint64_t *kp = nullptr, *ka = nullptr, *ki = nullptr, *kp2 = nullptr, *ka2 = nullptr,
           *ki2 = nullptr;
  int64_t *idx = nullptr, *idx2 = nullptr;
  unsigned long long* err = nullptr;       // [0] missing deadline, [1] NaN key, [2] keys sorted (device)
  unsigned long long* err_host = nullptr;  // pinned readback
  int policy = 0;
  const int64_t* last_ids = nullptr;  // device ids of the last scored queue (messages)
  // host-variant staging
  void* qdev = nullptr;
  double* outdev = nullptr;
  void* qhost = nullptr;    // pinned pack of the caller's queue arrays
  void* outhost = nullptr;  // pinned results before they are unpacked to the caller
  int64_t host_cap = 0;     // capacity of the four blocks above, in requests
};

namespace {

void scorer_free(tsb_scorer* s) {
  if (!s) return;
  cudaFree(s->kp);
  cudaFree(s->ka);
  cudaFree(s->ki);
  cudaFree(s->kp2);
  cudaFree(s->ka2);
  cudaFree(s->ki2);
  cudaFree(s->idx);
  cudaFree(s->idx2);
  cudaFree(s->err);
  cudaFreeHost(s->err_host);
  cudaFree(s->qdev);
  cudaFree(s->outdev);
  cudaFreeHost(s->qhost);
  cudaFreeHost(s->outhost);
}

tsb_status scorer_reserve(tsb_scorer* s, int64_t n) {
  if (n <= s->capacity) return TSB_OK;
  const int64_t cap = std::max<int64_t>(n, 1024);
  s->capacity = 0;  // a failed grow leaves no dangling buffer (scorer_free frees what is set)
  for (uint64_t** p : {&s->kp, &s->ka, &s->ki, &s->kp2, &s->ka2, &s->ki2}) {
    cudaFree(*p);
    *p = nullptr;
    TSB_CUDA_TRY(cudaMalloc(p, sizeof(uint64_t) * cap));
  }
  for (int64_t** p : {&s->idx, &s->idx2}) {
    cudaFree(*p);
    *p = nullptr;
    TSB_CUDA_TRY(cudaMalloc(p, sizeof(int64_t) * cap));
  }
  s->capacity = cap;
  return TSB_OK;
}

// Maps the K4 error words (already in err_host) to the reference's exceptions:
// MissingDeadline "<policy>: request <id> has no deadline" (scheduler.cpp:62-68).
tsb_status scorer_errors_from_host(tsb_scorer* s, int64_t* err_index) {
  const unsigned long long miss = s->err_host[0], nan = s->err_host[1];
  if (err_index) *err_index = -1;
  if (miss == ~0ull && nan == ~0ull) return TSB_OK;
  const unsigned long long first = std::min(miss, nan);
  if (err_index) *err_index = static_cast<int64_t>(first);
  int64_t id = 0;
  if (s->last_ids)
    TSB_CUDA_TRY(cudaMemcpy(&id, s->last_ids + first, sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (first == miss) {
    const char* pol = s->policy == TSB_EDF ? "edf" : "lstf";
    return fail(TSB_MISSING_DEADLINE,
                std::string(pol) + ": request " + std::to_string(id) + " has no deadline");
  }
  return fail(TSB_VALIDATION,
              "request " + std::to_string(id) + ": priority key is NaN (non-finite cost inputs)");
}

// Reads the K4 error words back (synchronising on stream) and maps them.
tsb_status scorer_check_errors(tsb_scorer* s, cudaStream_t st, int64_t* err_index) {
  TSB_CUDA_TRY(cudaMemcpyAsync(s->err_host, s->err, 2 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, st));
  TSB_CUDA_TRY(cudaStreamSynchronize(st));
  return scorer_errors_from_host(s, err_index);
}

}  // namespace

extern "C" {

tsb_status tsb_scorer_create(int device, int64_t capacity, tsb_scorer** out) {
  tsb::DeviceGuard dg(device);
  auto* s = new tsb_scorer();
  s->device = device;
  cudaError_t e = cudaMalloc(&s->err, 3 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMallocHost(&s->err_host, 2 * sizeof(unsigned long long));
  if (e != cudaSuccess) {
    scorer_free(s);
    delete s;
    return tsb::cuda_fail(e, "tsb_scorer_create");
  }
  tsb_status st = scorer_reserve(s, capacity);
  if (st != TSB_OK) {
    scorer_free(s);
    delete s;
    return st;
  }
  *out = s;
  return TSB_OK;
}

void tsb_scorer_destroy(tsb_scorer* s) {
  if (!s) return;
  tsb::DeviceGuard dg(s ? s->device : -1);
  scorer_free(s);
  delete s;
}

tsb_status tsb_score_queue_device(tsb_scorer* s, void* stream, int64_t n, const tsb_queue* q,
                                  int policy, const double models[4], const tsb_cluster* c,
                                  double* t_load, double* t_comp, double* primary,
                                  int64_t* order, int64_t* err_index) {
  if (policy < TSB_FIFO || policy > TSB_LSTF) return fail(TSB_VALIDATION, "unknown policy");
  if (n < 0) return fail(TSB_VALIDATION, "score_queue: n must be >= 0");
  tsb::DeviceGuard dg(s ? s->device : -1);
  if (c->block_size_tokens < 1)
    return fail(TSB_VALIDATION, "cluster: block_size_tokens must be >= 1");
  TSB_TRY(scorer_reserve(s, n));
  auto st = static_cast<cudaStream_t>(stream);
  s->policy = policy;
  s->last_ids = q->id;
  TSB_CUDA_TRY(cudaMemsetAsync(s->err, 0xff, 3 * sizeof(unsigned long long), st));
  tsb::ScoreParams p{policy, models[0], models[1], models[2], models[3], c->compute_quadratic,
                     c->block_size_tokens};
  TSB_CUDA_TRY(tsb::launch_score(n, *q, p, t_load, t_comp, primary, s->kp, s->ka, s->ki, s->err,
                                 s->err + 1, st));
  if (order)
    TSB_CUDA_TRY(tsb::launch_order(n, s->kp, s->ka, s->ki, s->idx, s->kp2, s->ka2, s->ki2,
                                   s->idx2, order, s->err + 2, st));
  if (err_index) return scorer_check_errors(s, st, err_index);
  return TSB_OK;
}

tsb_status tsb_scorer_check(tsb_scorer* s, void* stream, int64_t* err_index) {
  tsb::DeviceGuard dg(s ? s->device : -1);
  return scorer_check_errors(s, static_cast<cudaStream_t>(stream), err_index);
}

tsb_status tsb_score_queue(tsb_scorer* s, void* stream, int64_t n, const tsb_queue* q,
                           int policy, const double models[4], const tsb_cluster* c,
                           double* t_load, double* t_comp, double* primary, int64_t* order) {
  auto st = static_cast<cudaStream_t>(stream);
  if (n == 0) return TSB_OK;
  tsb::DeviceGuard dg(s ? s->device : -1);
  // Pack the SoA queue into one device block: 7 x 8-byte arrays + flags.
  const size_t w = sizeof(int64_t) * static_cast<size_t>(n);
  if (n > s->host_cap) {  // grow-only buffers: no allocation (and no implicit sync) per call
    const int64_t cap = std::max<int64_t>(n, 4096);
    const size_t wc = sizeof(int64_t) * static_cast<size_t>(cap);
    cudaFree(s->qdev);
    cudaFree(s->outdev);
    cudaFreeHost(s->qhost);
    cudaFreeHost(s->outhost);
    s->qdev = nullptr;
    s->outdev = nullptr;
    s->qhost = s->outhost = nullptr;
    s->host_cap = 0;
    TSB_CUDA_TRY(cudaMalloc(&s->qdev, 8 * wc + static_cast<size_t>(cap)));
    TSB_CUDA_TRY(cudaMalloc(&s->outdev, 4 * wc));  // t_load | t_comp | primary | order
    TSB_CUDA_TRY(cudaMallocHost(&s->qhost, 8 * wc + static_cast<size_t>(cap)));
    TSB_CUDA_TRY(cudaMallocHost(&s->outhost, 4 * wc));
    s->host_cap = cap;
  }
  // The queue block is packed at the CURRENT n's stride so one H2D moves exactly 8*w+n bytes.
  auto* b = static_cast<uint8_t*>(s->qdev);
  auto* hb = static_cast<uint8_t*>(s->qhost);
  tsb::HostCopyTeam::get().run({{hb + 0 * w, q->id, w},
                                {hb + 1 * w, q->arrival, w},
                                {hb + 2 * w, q->context_tokens, w},
                                {hb + 3 * w, q->query_tokens, w},
                                {hb + 4 * w, q->cache_hit_ratio, w},
                                {hb + 5 * w, q->deadline, w},
                                {hb + 6 * w, q->measured_t_load, w},
                                {hb + 7 * w, q->measured_t_comp, w},
                                {hb + 8 * w, q->flags, static_cast<size_t>(n)}},
                               tsb::HostCopyTeam::PACK_NT);
  TSB_CUDA_TRY(cudaMemcpyAsync(b, hb, 8 * w + static_cast<size_t>(n), cudaMemcpyHostToDevice, st));
  tsb_queue dq;
  dq.id = reinterpret_cast<const int64_t*>(b + 0 * w);
  dq.arrival = reinterpret_cast<const double*>(b + 1 * w);
  dq.context_tokens = reinterpret_cast<const int64_t*>(b + 2 * w);
  dq.query_tokens = reinterpret_cast<const int64_t*>(b + 3 * w);
  dq.cache_hit_ratio = reinterpret_cast<const double*>(b + 4 * w);
  dq.deadline = reinterpret_cast<const double*>(b + 5 * w);
  dq.measured_t_load = reinterpret_cast<const double*>(b + 6 * w);
  dq.measured_t_comp = reinterpret_cast<const double*>(b + 7 * w);
  dq.flags = b + 8 * w;
  double* o = s->outdev;
  auto* ord = reinterpret_cast<int64_t*>(o + 3 * n);
  // Scoring, the error words and the requested outputs in one stream pass: a single sync.
  TSB_TRY(tsb_score_queue_device(s, stream, n, &dq, policy, models, c, o, o + n, o + 2 * n, ord,
                                 nullptr));
  TSB_CUDA_TRY(cudaMemcpyAsync(s->err_host, s->err, 2 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, st));
  // Read back only the requested outputs: the three cost/key arrays are contiguous.
  auto* ho = static_cast<uint8_t*>(s->outhost);
  const int first = t_load ? 0 : t_comp ? 1 : primary ? 2 : 3;
  const int last = order ? 3 : primary ? 2 : t_comp ? 1 : t_load ? 0 : -1;
  if (last >= 0)
    TSB_CUDA_TRY(cudaMemcpyAsync(ho + first * w, o + first * n, (last - first + 1) * w,
                                 cudaMemcpyDeviceToHost, st));
  TSB_CUDA_TRY(cudaStreamSynchronize(st));
  TSB_TRY(scorer_errors_from_host(s, nullptr));
  std::vector<tsb::CopySpan> outs;
  void* dsts[4] = {t_load, t_comp, primary, order};
  for (int k = 0; k < 4; ++k)
    if (dsts[k]) outs.push_back({dsts[k], ho + k * w, w});
  tsb::HostCopyTeam::get().run(outs, tsb::HostCopyTeam::UNPACK_FLUSH);
  return TSB_OK;
}

// ---------------------------------------------------------------------------------------
// Prefix hasher (K3)
// ---------------------------------------------------------------------------------------
tsb_status tsb_hash_prefix_chunks_device(void* stream, int64_t n_req, const int64_t* offsets,
                                         const int32_t* tokens, const int64_t* chunk_offsets,
                                         uint64_t* out) {
  if (n_req < 0) return fail(TSB_VALIDATION, "hash_prefix_chunks: n_req must be >= 0");
  TSB_CUDA_TRY(tsb::launch_hash_prefix(n_req, offsets, tokens, chunk_offsets, out,
                                       static_cast<cudaStream_t>(stream)));
  return TSB_OK;
}

tsb_status tsb_hash_set_grid(int ctas_per_sm) {
  if (ctas_per_sm < 0 || ctas_per_sm > 8) return fail(TSB_VALIDATION, "hash_set_grid: 0..8 CTAs per SM");
  tsb::set_hash_grid(ctas_per_sm);
  return TSB_OK;
}

tsb_status tsb_hash_set_tuning(int prefetch_groups, int fused_chain) {
  if (prefetch_groups < -1 || prefetch_groups > 64) return fail(TSB_VALIDATION, "hash_set_tuning: prefetch 0..64 groups");
  if (fused_chain < -1 || fused_chain > 1) return fail(TSB_VALIDATION, "hash_set_tuning: fused_chain 0 or 1");
  if (prefetch_groups >= 0) tsb::set_hash_prefetch(prefetch_groups);
  if (fused_chain >= 0) tsb::set_hash_fused(fused_chain);
  return TSB_OK;
}

tsb_status tsb_hash_chunk_digests_device(void* stream, int64_t n_req, const int64_t* offsets,
                                         const int32_t* tokens, const int64_t* chunk_offsets, uint64_t* out) {
  if (n_req < 0) return fail(TSB_VALIDATION, "hash_chunk_digests: n_req must be >= 0");
  TSB_CUDA_TRY(tsb::launch_chunk_digests(n_req, offsets, tokens, chunk_offsets, out,
                                         static_cast<cudaStream_t>(stream)));
  return TSB_OK;
}

tsb_status tsb_hash_prefix_chunks(void* stream, int64_t n_req, const int64_t* offsets,
                                  const int32_t* tokens, uint64_t* out, int64_t* n_hashes) {
  auto st = static_cast<cudaStream_t>(stream);
  if (n_req < 0) return fail(TSB_VALIDATION, "hash_prefix_chunks: n_req must be >= 0");
  std::vector<int64_t> coff(static_cast<size_t>(n_req) + 1, 0);
  for (int64_t r = 0; r < n_req; ++r) {
    const int64_t len = offsets[r + 1] - offsets[r];
    if (len < 0) return fail(TSB_VALIDATION, "hash_prefix_chunks: offsets must be non-decreasing");
    coff[r + 1] = coff[r] + len / 256;
  }
  const int64_t total = coff[n_req];
  *n_hashes = total;
  if (total == 0) return TSB_OK;
  const int64_t ntok = offsets[n_req] - offsets[0];
  // Grow-only device buffers per (host thread, device): no cudaMalloc / cudaFree (and no implicit
  // device synchronisation) per call once the largest batch has been seen.
  int dev = 0;
  TSB_CUDA_TRY(cudaGetDevice(&dev));
  struct HashBufs {
    int64_t* off = nullptr;
    int64_t* coff = nullptr;
    int32_t* tok = nullptr;
    uint64_t* out = nullptr;
    int64_t n_req = 0, ntok = 0, total = 0;
  };
  thread_local std::vector<HashBufs> per_dev;
  if (static_cast<int>(per_dev.size()) <= dev) per_dev.resize(static_cast<size_t>(dev) + 1);
  HashBufs& b = per_dev[static_cast<size_t>(dev)];
  auto grow = [&](auto** p, int64_t& cap, int64_t need, size_t elem) -> cudaError_t {
    if (need <= cap) return cudaSuccess;
    cudaFree(*p);
    *p = nullptr;
    cap = 0;
    const int64_t n = std::max<int64_t>(need, cap + cap / 2);
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), elem * static_cast<size_t>(n));
    if (e == cudaSuccess) cap = n;
    return e;
  };
  int64_t n_cap = b.n_req, n_cap2 = b.n_req;
  cudaError_t e = grow(&b.off, n_cap, n_req + 1, sizeof(int64_t));
  if (e == cudaSuccess) e = grow(&b.coff, n_cap2, n_req + 1, sizeof(int64_t));
  if (e == cudaSuccess) b.n_req = std::min(n_cap, n_cap2);
  if (e == cudaSuccess) e = grow(&b.tok, b.ntok, std::max<int64_t>(ntok, 1), sizeof(int32_t));
  if (e == cudaSuccess) e = grow(&b.out, b.total, total, sizeof(uint64_t));
  if (e == cudaSuccess) {
    std::vector<int64_t> rel(offsets, offsets + n_req + 1);
    for (auto& v : rel) v -= offsets[0];
    e = cudaMemcpyAsync(b.off, rel.data(), sizeof(int64_t) * (n_req + 1), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(b.coff, coff.data(), sizeof(int64_t) * (n_req + 1), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(b.tok, tokens + offsets[0], sizeof(int32_t) * ntok, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = tsb::launch_hash_prefix(n_req, b.off, b.tok, b.coff, b.out, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(out, b.out, sizeof(uint64_t) * total, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  if (e != cudaSuccess) return tsb::cuda_fail(e, "tsb_hash_prefix_chunks");
  return TSB_OK;
}

tsb_status tsb_gen_tokens_device(void* stream, uint64_t seed, int64_t n_req,
                                 const int64_t* offsets, const int64_t* doc,
                                 const int64_t* shared_len, int32_t* out) {
  TSB_CUDA_TRY(tsb::launch_gen_tokens(seed, n_req, offsets, doc, shared_len, out,
                                      static_cast<cudaStream_t>(stream)));
  return TSB_OK;
}

}  // extern "C"
