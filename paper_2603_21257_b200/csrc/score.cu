// score.cu — K4 batched service-cost scorer and K5 schedule order for sm_100a.
//
// K4 restates estimate_service_cost (cost_model.cpp:56-71) + priority_key (scheduler.cpp:39-73)
// one thread per request, in f64 with explicitly rounded non-fused operations
// (__dmul_rn/__dadd_rn/__ddiv_rn) in the reference's evaluation order, so the scores are
// bit-identical to the reference built without FMA contraction.
//
// K5 replaces the O(N^2) pick_next drain (scheduler.cpp:75-100) with a sort under
// PriorityKey::operator< (scheduler.hpp:38-42).  Keys ignore `now` (scheduler.cpp:47), so for
// a fixed queue the drain order IS the sorted order.  Keys are encoded as order-preserving
// u64 triples (primary, arrival, id); -0.0 is canonicalised to +0.0 (equal under operator<).
// Sort = bitonic sort of 2048-key tiles in shared memory, then stable merge passes in which
// each element finds its output slot by binary search in the sibling run.  Latency-bound at
// 100K requests (~3 MB of keys): the point is microseconds instead of the CPU's milliseconds.
#include "common.cuh"
#include "kernels.h"

namespace tsb {
namespace {

__device__ __forceinline__ uint64_t enc_f64(double x) {
  x = __dadd_rn(x, 0.0);  // -0.0 -> +0.0 under round-to-nearest
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ uint64_t enc_i64(int64_t v) {
  return static_cast<uint64_t>(v) ^ 0x8000000000000000ull;
}

__global__ void k_score(int64_t n, tsb_queue q, ScoreParams p, double* __restrict__ t_load,
                        double* __restrict__ t_comp, double* __restrict__ primary,
                        uint64_t* __restrict__ kp, uint64_t* __restrict__ ka,
                        uint64_t* __restrict__ ki, unsigned long long* err_missing,
                        unsigned long long* err_nan) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint8_t fl = q.flags[i];
  const int64_t ctx = q.context_tokens[i];
  const double hit = q.cache_hit_ratio[i];
  double tl = 0.0, tc = 0.0;
  if (fl & TSB_HAS_MEASURED) {  // measured override returned verbatim (cost_model.cpp:58-59)
    tl = q.measured_t_load[i];
    tc = q.measured_t_comp[i];
  } else {
    // cached_token_count (types.cpp:73-79)
    const double hit_tokens = __dmul_rn(__ll2double_rn(ctx), hit);
    const int64_t blocks = __double2ll_rz(floor(__ddiv_rn(hit_tokens, __ll2double_rn(p.block))));
    const int64_t cached = blocks * p.block;
    // predict (cost_model.cpp:52-54): intercept + slope * tokens
    if (cached > 0) tl = __dadd_rn(p.load_icpt, __dmul_rn(p.load_slope, __ll2double_rn(cached)));
    const int64_t ct = ctx + q.query_tokens[i] - cached;  // types.cpp:81-83
    tc = __dadd_rn(p.comp_icpt, __dmul_rn(p.comp_slope, __ll2double_rn(ct)));
    if (p.quadratic > 0.0) {  // cost_model.cpp:66-69
      const double d = __ll2double_rn(ct);
      tc = __dadd_rn(tc, __dmul_rn(__dmul_rn(p.quadratic, d), d));
    }
  }
  const double arrival = q.arrival[i];
  double key = 0.0;
  switch (p.policy) {
    case TSB_FIFO: key = arrival; break;
    case TSB_SJF_PT: {  // prefill_token_estimate (scheduler.cpp:39-43)
      const double hit_tok = floor(__dmul_rn(__ll2double_rn(ctx), hit));
      key = __dsub_rn(__ll2double_rn(ctx + q.query_tokens[i]), hit_tok);
      break;
    }
    case TSB_SJF_COST: key = __dadd_rn(tl, tc); break;
    case TSB_EDF:
      if (!(fl & TSB_HAS_DEADLINE)) atomicMin(err_missing, static_cast<unsigned long long>(i));
      key = q.deadline[i];
      break;
    case TSB_LSTF:
      if (!(fl & TSB_HAS_DEADLINE)) atomicMin(err_missing, static_cast<unsigned long long>(i));
      key = __dsub_rn(q.deadline[i], __dadd_rn(tl, tc));
      break;
    default: break;
  }
  if (isnan(key) || isnan(arrival)) atomicMin(err_nan, static_cast<unsigned long long>(i));
  if (t_load) t_load[i] = tl;
  if (t_comp) t_comp[i] = tc;
  if (primary) primary[i] = key;
  kp[i] = enc_f64(key);
  ka[i] = enc_f64(arrival);
  ki[i] = enc_i64(q.id[i]);
}

struct Key {
  uint64_t p, a, i;
};

__device__ __forceinline__ bool key_less(const Key& x, const Key& y) {
  if (x.p != y.p) return x.p < y.p;
  if (x.a != y.a) return x.a < y.a;
  return x.i < y.i;
}

constexpr int kTile = 2048;
constexpr int kTileThreads = 1024;

// Bitonic sort of one tile in shared memory; pads with +inf keys.
__global__ void __launch_bounds__(kTileThreads) k_tile_sort(
    int64_t n, const uint64_t* __restrict__ kp, const uint64_t* __restrict__ ka,
    const uint64_t* __restrict__ ki, uint64_t* __restrict__ okp, uint64_t* __restrict__ oka,
    uint64_t* __restrict__ oki, int64_t* __restrict__ oidx, int64_t* __restrict__ order_out) {
  extern __shared__ __align__(16) uint64_t tile_smem[];
  uint64_t* sp = tile_smem;
  uint64_t* sa = sp + kTile;
  uint64_t* si = sa + kTile;
  int32_t* sx = reinterpret_cast<int32_t*>(si + kTile);
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
  for (int t = threadIdx.x; t < kTile; t += kTileThreads) {
    const int64_t g = base + t;
    if (g < n) {
      sp[t] = kp[g];
      sa[t] = ka[g];
      si[t] = ki[g];
    } else {
      sp[t] = sa[t] = si[t] = ~0ull;
    }
    sx[t] = t;
  }
  __syncthreads();
  for (int k = 2; k <= kTile; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int t = threadIdx.x;
      const int lo = 2 * t - (t & (j - 1));  // index with bit j clear
      const int hi = lo + j;
      const bool up = (lo & k) == 0;
      const Key x{sp[lo], sa[lo], si[lo]};
      const Key y{sp[hi], sa[hi], si[hi]};
      // Ties (duplicate keys) keep the lower original index first: stable.
      const bool gt = key_less(y, x) || (!key_less(x, y) && sx[lo] > sx[hi]);
      if (gt == up) {
        sp[lo] = y.p; sa[lo] = y.a; si[lo] = y.i;
        sp[hi] = x.p; sa[hi] = x.a; si[hi] = x.i;
        const int32_t tx = sx[lo];
        sx[lo] = sx[hi];
        sx[hi] = tx;
      }
      __syncthreads();
    }
  }
  for (int t = threadIdx.x; t < kTile; t += kTileThreads) {
    const int64_t g = base + t;
    if (g < n) {
      if (order_out) {
        order_out[g] = base + sx[t];
      } else {
        okp[g] = sp[t];
        oka[g] = sa[t];
        oki[g] = si[t];
        oidx[g] = base + sx[t];
      }
    }
  }
}

// One stable merge pass of runs of `width`: element e of run A lands at
// (e - startA) + #{b in B : b < e}; element of run B at (e - startB) + #{a in A : a <= e}.
__global__ void k_merge_pass(int64_t n, int64_t width, const uint64_t* __restrict__ kp,
                             const uint64_t* __restrict__ ka, const uint64_t* __restrict__ ki,
                             const int64_t* __restrict__ idx, uint64_t* __restrict__ okp,
                             uint64_t* __restrict__ oka, uint64_t* __restrict__ oki,
                             int64_t* __restrict__ oidx, int64_t* __restrict__ order_out) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= n) return;
  const int64_t pair_base = (e / (2 * width)) * (2 * width);
  const int64_t mid = min(pair_base + width, n);
  const int64_t end = min(pair_base + 2 * width, n);
  const bool in_a = e < mid;
  const Key x{kp[e], ka[e], ki[e]};
  int64_t lo = in_a ? mid : pair_base;
  int64_t hi = in_a ? end : mid;
  // lower_bound (A side counts strictly-less B keys) / upper_bound (B counts <= A keys)
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    const Key y{kp[m], ka[m], ki[m]};
    const bool go_right = in_a ? key_less(y, x) : !key_less(x, y);
    if (go_right) lo = m + 1;
    else hi = m;
  }
  const int64_t other_start = in_a ? mid : pair_base;
  const int64_t own_start = in_a ? pair_base : mid;
  const int64_t dst = pair_base + (e - own_start) + (lo - other_start);
  if (order_out) {
    order_out[dst] = idx[e];
  } else {
    okp[dst] = x.p;
    oka[dst] = x.a;
    oki[dst] = x.i;
    oidx[dst] = idx[e];
  }
}

}  // namespace

cudaError_t launch_score(int64_t n, tsb_queue q, ScoreParams p, double* t_load, double* t_comp,
                         double* primary, uint64_t* kp, uint64_t* ka, uint64_t* ki,
                         unsigned long long* err_missing, unsigned long long* err_nan,
                         cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_score<<<ceil_div(n, 256), 256, 0, st>>>(n, q, p, t_load, t_comp, primary, kp, ka, ki,
                                            err_missing, err_nan);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_order(int64_t n, uint64_t* kp, uint64_t* ka, uint64_t* ki, int64_t* idx,
                         uint64_t* kp2, uint64_t* ka2, uint64_t* ki2, int64_t* idx2,
                         int64_t* order_out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int tiles = ceil_div(n, kTile);
  constexpr size_t kTileSmem = kTile * (3 * sizeof(uint64_t) + sizeof(int32_t));
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_tile_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kTileSmem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (tiles == 1) {
    k_tile_sort<<<1, kTileThreads, kTileSmem, st>>>(n, kp, ka, ki, nullptr, nullptr, nullptr, nullptr,
                                            order_out);
    count_launch();
    return cudaGetLastError();
  }
  k_tile_sort<<<tiles, kTileThreads, kTileSmem, st>>>(n, kp, ka, ki, kp2, ka2, ki2, idx2, nullptr);
  count_launch();
  uint64_t *sp = kp2, *sa = ka2, *si = ki2, *dp = kp, *da = ka, *di = ki;
  int64_t *sx = idx2, *dx = idx;
  for (int64_t width = kTile; width < n; width *= 2) {
    const bool last = width * 2 >= n;
    k_merge_pass<<<ceil_div(n, 256), 256, 0, st>>>(n, width, sp, sa, si, sx, dp, da, di, dx,
                                                   last ? order_out : nullptr);
    count_launch();
    std::swap(sp, dp);
    std::swap(sa, da);
    std::swap(si, di);
    std::swap(sx, dx);
  }
  return cudaGetLastError();
}

}  // namespace tsb
