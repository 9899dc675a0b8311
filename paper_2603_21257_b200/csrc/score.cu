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
// u64 triples (primary, arrival, id); -0.0 is canonicalised to +0.0 (equal under operator<); the
// original queue index breaks any remaining tie (first-minimum wins, scheduler.cpp:85).
// Sort = merge sort: each 512-thread CTA sorts a 2048-record tile (4 records per thread sorted
// by a register network, then 9 merge-path rounds in shared memory), then one merge-path pass
// per doubling of the run width, in which every CTA produces 1024 outputs: one warp finds each
// end of the CTA's output window with a 32-ary search over global memory, the window's inputs
// are staged in shared memory, and each thread merges 4 outputs.  Latency-bound at 100K
// requests (~3 MB of keys).
#include <algorithm>

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

// ---- K5 -----------------------------------------------------------------------------------------
struct Rec {
  uint64_t p, a, i;
  int64_t x;  // original queue index
};

__device__ __forceinline__ bool rec_less(const Rec& u, const Rec& v) {
  if (u.p != v.p) return u.p < v.p;
  if (u.a != v.a) return u.a < v.a;
  if (u.i != v.i) return u.i < v.i;
  return u.x < v.x;
}

__device__ __forceinline__ void cswap(Rec& u, Rec& v) {
  if (rec_less(v, u)) {
    const Rec t = u;
    u = v;
    v = t;
  }
}

constexpr int kItems = 4;
constexpr int kThreads = 512;
constexpr int kTileN = kItems * kThreads;  // 2048 records per tile-sort CTA
constexpr int kMergeThreads = 256;
constexpr int kMergeN = kItems * kMergeThreads;  // 1024 outputs per merge-pass CTA
constexpr Rec kPad = {~0ull, ~0ull, ~0ull, 0x7fffffffffffffffll};

// Shared-memory record L lives at byte L*32 + (L/4)*8: the 8-byte pad after every 4 records
// makes both the blocked (thread t <-> records 4t..4t+3) and the striped (lane <-> record)
// access patterns 2-way instead of 32-way / 8-way bank-conflicted.
constexpr size_t smem_bytes(int n) { return static_cast<size_t>(n) * 32 + static_cast<size_t>(n / 4) * 8; }
__device__ __forceinline__ Rec& sat(uint8_t* sb, int L) {
  return *reinterpret_cast<Rec*>(sb + static_cast<size_t>(L) * 32 + static_cast<size_t>(L >> 2) * 8);
}

__device__ __forceinline__ Rec load_rec(const uint64_t* kp, const uint64_t* ka, const uint64_t* ki,
                                        const int64_t* idx, int64_t g) {
  return Rec{kp[g], ka[g], ki[g], idx ? idx[g] : g};
}

// Merge path inside shared memory (runs A = [a, a+alen), B = [b, b+blen) in record indices):
// number of A records among the first d merged outputs.
__device__ __forceinline__ int merge_path(uint8_t* sb, int a, int alen, int b, int blen, int d) {
  int lo = max(0, d - blen), hi = min(d, alen);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (rec_less(sat(sb, a + mid), sat(sb, b + d - 1 - mid))) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Serial merge of kItems outputs starting at A + ai, B + bi.
__device__ __forceinline__ void merge_items(uint8_t* sb, int a, int alen, int b, int blen, int ai,
                                            int bi, Rec (&r)[kItems]) {
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const bool take_a = bi >= blen || (ai < alen && rec_less(sat(sb, a + ai), sat(sb, b + bi)));
    r[k] = take_a ? sat(sb, a + ai++) : sat(sb, b + bi++);
  }
}

__global__ void __launch_bounds__(kThreads, 1) k_tile_sort(
    int64_t n, const uint64_t* __restrict__ kp, const uint64_t* __restrict__ ka,
    const uint64_t* __restrict__ ki, uint64_t* __restrict__ okp, uint64_t* __restrict__ oka,
    uint64_t* __restrict__ oki, int64_t* __restrict__ oidx, int64_t* __restrict__ order_out,
    const unsigned long long* __restrict__ sorted) {
  pdl_wait();
  if (*sorted) return;  // the queue is already in key order: k_iota_if_sorted writes the order
  extern __shared__ __align__(16) uint8_t sbuf[];
  const int t = threadIdx.x;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTileN;
  // striped (coalesced) load into shared memory, then each thread takes 4 consecutive records
  for (int e = t; e < kTileN; e += kThreads) {
    const int64_t g = base + e;
    sat(sbuf, e) = g < n ? load_rec(kp, ka, ki, nullptr, g) : kPad;
  }
  __syncthreads();
  Rec r[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) r[k] = sat(sbuf, t * kItems + k);
  // 4-record sorting network
  cswap(r[0], r[1]);
  cswap(r[2], r[3]);
  cswap(r[0], r[2]);
  cswap(r[1], r[3]);
  cswap(r[1], r[2]);
  for (int w = kItems; w < kTileN; w <<= 1) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kItems; ++k) sat(sbuf, t * kItems + k) = r[k];
    __syncthreads();
    const int start = (t * kItems) & ~(2 * w - 1);
    const int d = t * kItems - start;
    const int ai = merge_path(sbuf, start, w, start + w, w, d);
    merge_items(sbuf, start, w, start + w, w, ai, d - ai, r);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kItems; ++k) sat(sbuf, t * kItems + k) = r[k];
  __syncthreads();
  for (int e = t; e < kTileN; e += kThreads) {
    const int64_t g = base + e;
    if (g >= n) continue;
    const Rec v = sat(sbuf, e);
    if (order_out) {
      order_out[g] = v.x;
    } else {
      okp[g] = v.p;
      oka[g] = v.a;
      oki[g] = v.i;
      oidx[g] = v.x;
    }
  }
}

// 32-ary merge-path search over global memory by one warp: number of A records among the first
// d outputs of merge(A, B).
__device__ int warp_merge_path(const uint64_t* kp, const uint64_t* ka, const uint64_t* ki,
                               const int64_t* idx, int64_t a0, int64_t alen, int64_t b0,
                               int64_t blen, int64_t d) {
  const int lane = threadIdx.x & 31;
  int64_t lo = d - blen > 0 ? d - blen : 0, hi = d < alen ? d : alen;
  while (hi > lo) {
    const int64_t span = hi - lo;
    const int64_t step = span <= 32 ? 1 : (span + 31) / 32;
    const int64_t i = lo + lane * step;
    bool f = false;
    if (i < hi)
      f = rec_less(load_rec(kp, ka, ki, idx, a0 + i), load_rec(kp, ka, ki, idx, b0 + d - 1 - i));
    const unsigned b = __ballot_sync(0xffffffffu, f);
    const int k = __popc(b);
    if (step == 1) return static_cast<int>(lo + k);
    if (k == 0) return static_cast<int>(lo);
    const int64_t nlo = lo + (k - 1) * step + 1;
    const int64_t ik = lo + k * step;
    if (k < 32 && ik < hi) hi = ik;
    lo = nlo;
  }
  return static_cast<int>(lo);
}

__global__ void __launch_bounds__(kMergeThreads) k_merge_pass(
    int64_t n, int64_t width, const uint64_t* __restrict__ kp, const uint64_t* __restrict__ ka,
    const uint64_t* __restrict__ ki, const int64_t* __restrict__ idx, uint64_t* __restrict__ okp,
    uint64_t* __restrict__ oka, uint64_t* __restrict__ oki, int64_t* __restrict__ oidx,
    int64_t* __restrict__ order_out, const unsigned long long* __restrict__ sorted) {
  pdl_wait();
  if (*sorted) return;
  extern __shared__ __align__(16) uint8_t sbuf[];
  __shared__ int split[2];
  const int t = threadIdx.x, warp = t >> 5;
  const int64_t out_begin = static_cast<int64_t>(blockIdx.x) * kMergeN;
  const int64_t pair_base = (out_begin / (2 * width)) * (2 * width);
  const int64_t a0 = pair_base, alen = min(width, n - pair_base);
  const int64_t b0 = a0 + alen;
  const int64_t brem = n - b0 < width ? n - b0 : width;
  const int64_t blen = brem > 0 ? brem : 0;
  const int64_t d0 = out_begin - pair_base;
  const int64_t d1 = d0 + kMergeN < alen + blen ? d0 + kMergeN : alen + blen;
  if (warp < 2) {
    const int sp = warp_merge_path(kp, ka, ki, idx, a0, alen, b0, blen, warp == 0 ? d0 : d1);
    if ((t & 31) == 0) split[warp] = sp;
  }
  __syncthreads();
  const int s0 = split[0], s1 = split[1];
  const int wa = s1 - s0, wb = static_cast<int>((d1 - s1) - (d0 - s0));
  for (int e = t; e < wa + wb; e += kMergeThreads) {
    sat(sbuf, e) = e < wa ? load_rec(kp, ka, ki, idx, a0 + s0 + e)
                          : load_rec(kp, ka, ki, idx, b0 + (d0 - s0) + (e - wa));
  }
  __syncthreads();
  const int dt = t * kItems;
  const int total = wa + wb;
  if (dt < total) {
    const int ai = merge_path(sbuf, 0, wa, wa, wb, dt);
    Rec r[kItems];
    merge_items(sbuf, 0, wa, wa, wb, ai, dt - ai, r);
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      if (dt + k >= total) break;
      const int64_t g = pair_base + d0 + dt + k;
      if (order_out) {
        order_out[g] = r[k].x;
      } else {
        okp[g] = r[k].p;
        oka[g] = r[k].a;
        oki[g] = r[k].i;
        oidx[g] = r[k].x;
      }
    }
  }
}

// Adaptive fast path: a queue whose records are already in key order (FIFO over an arrival-
// ordered queue, the common case) needs no sort.  One pass clears *sorted on the first
// out-of-order neighbour pair; the sort kernels then run only if it was cleared, and
// k_iota_if_sorted writes the identity permutation otherwise.
__global__ void k_check_sorted(int64_t n, const uint64_t* __restrict__ kp,
                               const uint64_t* __restrict__ ka, const uint64_t* __restrict__ ki,
                               unsigned long long* __restrict__ sorted) {
  pdl_wait();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  bool ok = true;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i + 1 < n; i += stride)
    ok &= rec_less(load_rec(kp, ka, ki, nullptr, i), load_rec(kp, ka, ki, nullptr, i + 1));
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) *sorted = 0;
}

__global__ void k_iota_if_sorted(int64_t n, const unsigned long long* __restrict__ sorted,
                                 int64_t* __restrict__ order_out) {
  pdl_wait();
  if (!*sorted) return;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    order_out[i] = i;
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
                         int64_t* order_out, unsigned long long* sorted, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int check_grid = static_cast<int>(std::min<int64_t>(ceil_div(n, 256), 148 * 4));
  TSB_PDL(k_check_sorted, check_grid, 256, 0, st, n, kp, ka, ki, sorted);
  constexpr size_t kSmem = smem_bytes(kTileN);       // 68 KiB
  constexpr size_t kMergeSmem = smem_bytes(kMergeN);  // 34 KiB
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    cudaError_t e = cudaFuncSetAttribute(k_tile_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kSmem));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_merge_pass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(kMergeSmem));
    if (e != cudaSuccess) return e;
  }
  const int tiles = ceil_div(n, kTileN);
  if (tiles == 1) {
    TSB_PDL(k_tile_sort, 1, kThreads, kSmem, st, n, kp, ka, ki, nullptr, nullptr, nullptr, nullptr,
            order_out, sorted);
  } else {
  TSB_PDL(k_tile_sort, tiles, kThreads, kSmem, st, n, kp, ka, ki, kp2, ka2, ki2, idx2, nullptr, sorted);
  uint64_t *sp = kp2, *sa = ka2, *si = ki2, *dp = kp, *da = ka, *di = ki;
  int64_t *sx = idx2, *dx = idx;
  for (int64_t width = kTileN; width < n; width *= 2) {
    const bool last = width * 2 >= n;
    TSB_PDL(k_merge_pass, ceil_div(n, kMergeN), kMergeThreads, kMergeSmem, st, n, width,
            static_cast<const uint64_t*>(sp), static_cast<const uint64_t*>(sa),
            static_cast<const uint64_t*>(si), static_cast<const int64_t*>(sx), dp, da, di, dx,
            last ? order_out : nullptr, static_cast<const unsigned long long*>(sorted));
    std::swap(sp, dp);
    std::swap(sa, da);
    std::swap(si, di);
    std::swap(sx, dx);
  }
  }
  TSB_PDL(k_iota_if_sorted, check_grid, 256, 0, st, n, static_cast<const unsigned long long*>(sorted),
          order_out);
  return cudaGetLastError();
}

}  // namespace tsb
