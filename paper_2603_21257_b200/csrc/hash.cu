// hash.cu — K3 warp-parallel prefix chunk hasher (+ synthetic token generator) for sm_100a.
//
// The reference's only hash is byte-serial FNV-1a-64 (engine.cpp:500-507), used for a config
// fingerprint; it has no prefix hasher.  The definition frozen in
// oracle/tsb_oracle.c (orc_hash_prefix_chunks) keeps FNV-1a's constants and step, applied to
// 64-bit words (two int32 token ids each): 16 leaves of 8 words per 256-token chunk, a 4-level
// pairwise tree, and a per-request chain so hash c names the whole prefix [0, 256(c+1)).
//
// Mapping, two phases.  (1) k_chunk_digest: each warp of a persistent grid walks one contiguous,
// equal share of the global chunk index space (balanced however request lengths vary); each
// half-warp owns one chunk per round (lane j folds leaf j = words 32k+2j, 32k+2j+1 for k = 0..3, so each of the
// four 16-byte load instructions reads 2 x 256 contiguous bytes -- fully coalesced), two rounds
// are loaded before any is consumed (4 KiB in flight per warp), the tree is 4 shuffle levels
// inside the half-warp, and the digest goes to out[c].  (2) k_chain: one thread per request
// folds its digests into the chain in place (L2-resident).  HBM-bound: 4 B/token + 8 B/chunk.
#include "common.cuh"
#include "kernels.h"

namespace tsb {
namespace {

// One FNV step (h ^ w) * P with P = 2^40 + 0x1b3 (engine.cpp:504): in 32-bit halves the product
// is lo*0x1b3 (wide) with hi*0x1b3 + (lo << 8) added to the upper word -- three IMADs where the
// generic 64-bit multiply takes four.
__device__ __forceinline__ uint64_t fstep(uint64_t h, uint64_t w) {
  static_assert(kFnvPrime == (1ull << 40) + 0x1b3, "FNV-64 prime");
  const uint64_t x = h ^ w;
  uint64_t r;
  asm("{\n.reg .u32 xl, xh, rl, rh;\n"
      "mov.b64 {xl, xh}, %1;\n"
      "mul.wide.u32 %0, xl, 0x1b3;\n"
      "mov.b64 {rl, rh}, %0;\n"
      "mad.lo.u32 rh, xh, 0x1b3, rh;\n"
      "mad.lo.u32 rh, xl, 256, rh;\n"
      "mov.b64 %0, {rl, rh};\n}"
      : "=l"(r)
      : "l"(x));
  return r;
}
__device__ __forceinline__ uint64_t fpair(uint64_t a, uint64_t b) {
  return fstep(fstep(kFnvOffset, a), b);
}

constexpr int kHashThreads = 256;
constexpr int kHashWarps = kHashThreads / 32;

// Token ids are read exactly once: stream them through L2 with evict_first so the 87 MB of chunk
// digests written by phase 1 survive in L2 for phase 2.
__device__ __forceinline__ int4 ld_evict_first(const void* p) {
  int4 r;
  asm volatile(
      "{\n.reg .b64 pol;\n"
      "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], pol;\n}"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}

struct Leaf {
  int4 v[4];  // 16 int32 tokens
};

// Lane j of a half-warp loads tokens [64k + 4j, 64k + 4j + 4) for k = 0..3: every 16-byte load
// instruction of the warp reads two contiguous 256-byte runs (one per chunk).
__device__ __forceinline__ int2 ld_evict_first2(const void* p) {
  int2 r;
  asm volatile(
      "{\n.reg .b64 pol;\n"
      "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0,%1}, [%2], pol;\n}"
      : "=r"(r.x), "=r"(r.y)
      : "l"(p));
  return r;
}

// Token bases are 4-byte aligned only (requests have arbitrary lengths): 16-byte loads when the
// leaf's address allows, else 8-byte, else 4-byte (the class is uniform over a half-warp).
__device__ __forceinline__ void load_leaf(const int32_t* p, Leaf& f) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  if ((a & 15) == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) f.v[k] = ld_evict_first(p + 64 * k);
  } else if ((a & 7) == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int2 lo = ld_evict_first2(p + 64 * k), hi = ld_evict_first2(p + 64 * k + 2);
      f.v[k] = make_int4(lo.x, lo.y, hi.x, hi.y);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      f.v[k] = make_int4(__ldg(p + 64 * k), __ldg(p + 64 * k + 1), __ldg(p + 64 * k + 2),
                         __ldg(p + 64 * k + 3));
  }
}

__device__ __forceinline__ uint64_t word(int lo, int hi) {
  return static_cast<uint64_t>(static_cast<uint32_t>(lo)) |
         (static_cast<uint64_t>(static_cast<uint32_t>(hi)) << 32);
}

__device__ __forceinline__ uint64_t fold_leaf(const Leaf& f) {
  uint64_t h = kFnvOffset;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    h = fstep(h, word(f.v[k].x, f.v[k].y));
    h = fstep(h, word(f.v[k].z, f.v[k].w));
  }
  return h;
}

// Phase 1 -- chunk digests, balanced over the GLOBAL chunk index space (request lengths vary
// 100x, so a warp-per-request mapping leaves a long tail).  Each CTA of the persistent grid owns
// one contiguous, equal share of the chunk index space, which its warps walk interleaved: a warp
// finds its first chunk's request once (32-ary search over chunk_offsets) and then walks
// forward, each half-warp carrying its own (request, chunk base, token base) and stepping to the
// next request only at a boundary (~once per 100 chunks).  No per-chunk lookups sit between the
// token loads.
//
// Measured variants are in profiles/r01_k3_variants.md: TMA / cp.async staging with a
// lane-per-chunk fold (5x fewer instructions) lost to instruction-cache misses, bank conflicts
// of 1 KiB-strided chunks, and per-copy TMA cost (2.3-5.1 ms).
__device__ __forceinline__ void st_evict_last(uint64_t* p, uint64_t v) {
  asm volatile(
      "{\n.reg .b64 pol;\n"
      "createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
      "st.global.L2::cache_hint.b64 [%0], %1, pol;\n}" ::"l"(p),
      "l"(v)
      : "memory");
}

__device__ __forceinline__ int64_t warp_upper_bound(const int64_t* __restrict__ a, int64_t n,
                                                    int64_t v) {
  // first index i in [0, n) with a[i] > v (a non-decreasing), by 32-ary narrowing
  const int lane = threadIdx.x & 31;
  int64_t lo = 0, hi = n;
  while (hi > lo) {
    const int64_t span = hi - lo;
    const int64_t step = span <= 32 ? 1 : (span + 31) / 32;
    const int64_t i = lo + lane * step;
    const bool le = i < hi && a[i] <= v;
    const int k = __popc(__ballot_sync(0xffffffffu, le));
    if (step == 1) return lo + k;
    if (k == 0) return lo;
    const int64_t nlo = lo + (k - 1) * step + 1;
    if (k < 32 && lo + k * step < hi) hi = lo + k * step;
    lo = nlo;
  }
  return lo;
}

// Running position of one half-warp: the request owning chunk `c` and its bases.
struct ReqCursor {
  int64_t r, cb, nb, tb;  // request, its first chunk, next request's first chunk, token base
  __device__ __forceinline__ int64_t base_of(int64_t c, const int64_t* __restrict__ co,
                                             const int64_t* __restrict__ offs) {
    while (c >= nb) {  // rare: crossing into the next non-empty request
      ++r;
      cb = nb;
      nb = co[r + 1];
      tb = offs[r];
    }
    return tb + (c - cb) * 256;
  }
};

// The 4-level pairwise tree of two rounds at once (leaf j of round 0 in v0, of round 1 in v1, on
// lane j of each half-warp).  Level 1 pairs round 0 on even lanes and round 1 on odd lanes, so
// levels 2-4 carry both rounds in one shuffle + FNV pair per lane instead of two.  Round 0's
// digest ends in lane 0, round 1's in lane 1.
__device__ __forceinline__ uint64_t tree16x2(uint64_t v0, uint64_t v1, int j) {
  const uint64_t r = __shfl_xor_sync(0xffffffffu, (j & 1) ? v0 : v1, 1, 16);
  uint64_t v = (j & 1) ? fpair(r, v1) : fpair(v0, r);
#pragma unroll
  for (int d = 2; d < 16; d <<= 1) {
    const uint64_t o = __shfl_down_sync(0xffffffffu, v, d, 16);
    if ((j & (2 * d - 1)) < 2) v = fpair(v, o);
  }
  return v;
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Per-lane request search (one-time, for the prefetch cursor): first r with co[r + 1] > c.
__device__ __forceinline__ int64_t lane_request_of(const int64_t* __restrict__ co, int64_t n_req,
                                                   int64_t c) {
  int64_t lo = 0, hi = n_req;  // answer in [lo, hi)
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (co[mid] <= c) lo = mid; else hi = mid;
  }
  return lo;
}

// Rotating software pipeline of two rounds: the loads of round u + 2 are issued as soon as round
// u has been folded, so a warp keeps 1-2 rounds (2 KiB each) in flight while it computes.  With
// pf > 0 every lane also prefetches one 128-byte line of the warp's group pf iterations ahead
// into L2 (32 lines = the group's 4 chunks), so the loads hit L2 and more bytes are in flight
// than the registers hold.
template <bool kPf>
__device__ __forceinline__ void digest_range(int64_t n_req, const int64_t* __restrict__ offsets,
                                             const int32_t* __restrict__ tokens,
                                             const int64_t* __restrict__ chunk_offsets,
                                             uint64_t* __restrict__ out, int pf, int64_t total,
                                             int64_t c_begin, int64_t c_end) {
  const int lane = threadIdx.x & 31;
  const int half = lane >> 4, j = lane & 15;
  // The CTA owns a contiguous, equal share of the chunk space; its 8 warps interleave over it in
  // groups of 4 chunks (2 rounds x 2 half-warps), so each CTA streams one region with all its
  // warps on adjacent addresses.
  const int w = threadIdx.x >> 5;
  const int64_t first = c_begin + 4 * w;
  if (first >= c_end) return;
  constexpr int64_t kStride = 4 * kHashWarps;  // chunks between a warp's consecutive groups
  ReqCursor cur;
  cur.r = warp_upper_bound(chunk_offsets, n_req + 1, first) - 1;
  cur.cb = chunk_offsets[cur.r];
  cur.nb = chunk_offsets[cur.r + 1];
  cur.tb = offsets[cur.r];
  // prefetch cursor: lane l covers line (l & 7) of chunk (l >> 3) of the group pf iterations on
  const int64_t pf_off = static_cast<int64_t>(pf) * kStride + (lane >> 3);
  ReqCursor pcur;
  if (kPf) {
    const int64_t pc = min(first + pf_off, total - 1);
    pcur.r = lane_request_of(chunk_offsets, n_req, pc);
    pcur.cb = chunk_offsets[pcur.r];
    pcur.nb = chunk_offsets[pcur.r + 1];
    pcur.tb = offsets[pcur.r];
  }
  Leaf f[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int64_t cc = first + 2 * u + half;
    if (cc < c_end) {
      const int64_t base = cur.base_of(cc, chunk_offsets, offsets);
      load_leaf(tokens + base + j * 4, f[u]);
    }
  }
  for (int64_t c = first; c < c_end; c += kStride) {
    if (kPf) {
      const int64_t pc = c + pf_off;
      if (pc < c_end) prefetch_l2(tokens + pcur.base_of(pc, chunk_offsets, offsets) + (lane & 7) * 32);
    }
    uint64_t v[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      v[u] = fold_leaf(f[u]);
      const int64_t nc = c + 2 * u + half + kStride;
      if (nc < c_end) {
        const int64_t base = cur.base_of(nc, chunk_offsets, offsets);
        load_leaf(tokens + base + j * 4, f[u]);
      }
    }
    const uint64_t d = tree16x2(v[0], v[1], j);
    const int64_t cc = c + 2 * j + half;  // lane 0: round 0's chunk, lane 1: round 1's
    if (j < 2 && cc < c_end) st_evict_last(out + cc, d);  // keep digests in L2 for the chain
  }
}

template <bool kPf>
__global__ void __launch_bounds__(kHashThreads, 3) k_chunk_digest(
    int64_t n_req, const int64_t* __restrict__ offsets, const int32_t* __restrict__ tokens,
    const int64_t* __restrict__ chunk_offsets, uint64_t* __restrict__ out, int pf) {
  const int64_t total = chunk_offsets[n_req];
  const int64_t c_begin = total * blockIdx.x / gridDim.x;
  const int64_t c_end = total * (blockIdx.x + 1) / gridDim.x;
  digest_range<kPf>(n_req, offsets, tokens, chunk_offsets, out, pf, total, c_begin, c_end);
}

// ---- Phases 1 + 2 in one kernel -------------------------------------------------------------
// The CTA's 8 digest warps hand each iteration's 32 consecutive digests to a 9th warp through a
// shared-memory ring (an mbarrier pair per slot, 16 slots); the chain warp folds them into the
// per-request chain in chunk order while the digest warps stream on, and writes the chained
// hashes (one coalesced 256-byte store per iteration).  A request that began in an earlier CTA's
// range has no known chain value there, so its digests are written raw; k_chain_tail continues
// those few requests (at most one per range boundary) from the chained value the previous CTA
// wrote at its range end.
constexpr int kRing = 16;
constexpr int kFusedThreads = kHashThreads + 32;
constexpr uint64_t kChainInit = (kFnvOffset << 32) | (kFnvOffset >> 32);

// ring slot s: full[s] completes when the 8 digest warps have written it (one arrival each),
// empty[s] when the chain warp has consumed it; parity = (iteration / kRing) & 1.
struct RingBars {
  uint64_t full[kRing];
  uint64_t empty[kRing];
};

template <bool kPf>
__device__ __forceinline__ void digest_warp_ring(int64_t n_req, const int64_t* __restrict__ offsets,
                                                 const int32_t* __restrict__ tokens,
                                                 const int64_t* __restrict__ chunk_offsets, int pf,
                                                 int64_t total, int64_t c_begin, int64_t c_end,
                                                 int64_t iters, uint64_t (*ring)[32],
                                                 RingBars& bars) {
  const int lane = threadIdx.x & 31;
  const int half = lane >> 4, j = lane & 15;
  const int w = threadIdx.x >> 5;
  constexpr int64_t kStride = 4 * kHashWarps;
  const int64_t first = c_begin + 4 * w;
  const bool any = first < c_end;
  ReqCursor cur, pcur;
  const int64_t pf_off = static_cast<int64_t>(pf) * kStride + (lane >> 3);
  Leaf f[2];
  if (any) {
    cur.r = warp_upper_bound(chunk_offsets, n_req + 1, first) - 1;
    cur.cb = chunk_offsets[cur.r];
    cur.nb = chunk_offsets[cur.r + 1];
    cur.tb = offsets[cur.r];
    if (kPf) {
      const int64_t pc = min(first + pf_off, total - 1);
      pcur.r = lane_request_of(chunk_offsets, n_req, pc);
      pcur.cb = chunk_offsets[pcur.r];
      pcur.nb = chunk_offsets[pcur.r + 1];
      pcur.tb = offsets[pcur.r];
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t cc = first + 2 * u + half;
      if (cc < c_end) load_leaf(tokens + cur.base_of(cc, chunk_offsets, offsets) + j * 4, f[u]);
    }
  }
  for (int64_t i = 0; i < iters; ++i) {
    const int64_t c = first + i * kStride;
    const int slot = static_cast<int>(i % kRing);
    uint64_t d = 0;
    if (c < c_end) {
      if (kPf) {
        const int64_t pc = c + pf_off;
        if (pc < c_end) prefetch_l2(tokens + pcur.base_of(pc, chunk_offsets, offsets) + (lane & 7) * 32);
      }
      uint64_t v[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        v[u] = fold_leaf(f[u]);
        const int64_t nc = c + 2 * u + half + kStride;
        if (nc < c_end) load_leaf(tokens + cur.base_of(nc, chunk_offsets, offsets) + j * 4, f[u]);
      }
      d = tree16x2(v[0], v[1], j);
    }
    if (i >= kRing) mbar_wait(&bars.empty[slot], static_cast<uint32_t>((i / kRing - 1) & 1));
    if (j < 2) ring[slot][4 * w + 2 * j + half] = d;  // chunk c + 2j + half of this iteration
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars.full[slot]);
  }
}

__device__ __forceinline__ void chain_warp_ring(int64_t n_req, const int64_t* __restrict__ co,
                                                uint64_t* __restrict__ out, int64_t c_begin,
                                                int64_t c_end, int64_t iters,
                                                uint64_t (*ring)[32], RingBars& bars) {
  const int lane = threadIdx.x & 31;
  int64_t r = 0, nb = 0, nnb = 0;
  bool active = false;
  if (c_begin < c_end) {
    r = warp_upper_bound(co, n_req + 1, c_begin) - 1;
    active = co[r] >= c_begin;  // else the request began in an earlier range: raw digests
    nb = co[r + 1];
    nnb = co[min(r + 2, n_req)];
  }
  uint64_t h = kChainInit;
  for (int64_t i = 0; i < iters; ++i) {
    const int slot = static_cast<int>(i % kRing);
    const int64_t base = c_begin + i * 32;
    const int n = static_cast<int>(min(c_end - base, int64_t{32}));
    mbar_wait(&bars.full[slot], static_cast<uint32_t>((i / kRing) & 1));
    // bit k: a request begins at chunk base + k (nb is the next request's first chunk)
    uint32_t starts = 0;
    while (nb < base + n) {
      starts |= 1u << static_cast<int>(nb - base);
      ++r;
      nb = nnb;
      nnb = co[min(r + 2, n_req)];
    }
    const uint64_t* row = ring[slot];
    uint64_t mine = row[lane];
    if (starts == 0 && n == 32) {
      // common case (~3 in 4 iterations): the whole iteration continues one request
      if (active) {
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          h = fpair(h, row[k]);
          mine = lane == k ? h : mine;
        }
      }
    } else {
      // branch-free: restart the chain at every request start, stop at n
      bool act = active;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const uint64_t d = row[k];
        const bool st = (starts >> k) & 1u;
        h = st ? kChainInit : h;
        act = act || st;
        const uint64_t g = fpair(h, d);
        const bool use = act && k < n;
        h = use ? g : h;
        mine = lane == k ? (use ? g : d) : mine;
      }
      active = act;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars.empty[slot]);
    if (lane < n) out[base + lane] = mine;
  }
}

template <bool kPf>
__global__ void __launch_bounds__(kFusedThreads, 3) k_chunk_hash_fused(
    int64_t n_req, const int64_t* __restrict__ offsets, const int32_t* __restrict__ tokens,
    const int64_t* __restrict__ chunk_offsets, uint64_t* __restrict__ out, int pf) {
  __shared__ uint64_t ring[kRing][32];
  __shared__ RingBars bars;
  if (threadIdx.x == 0) {
    for (int k = 0; k < kRing; ++k) {
      mbar_init(&bars.full[k], kHashWarps);
      mbar_init(&bars.empty[k], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t total = chunk_offsets[n_req];
  const int64_t c_begin = total * blockIdx.x / gridDim.x;
  const int64_t c_end = total * (blockIdx.x + 1) / gridDim.x;
  const int64_t iters = (c_end - c_begin + 31) / 32;
  if ((threadIdx.x >> 5) == kHashWarps)
    chain_warp_ring(n_req, chunk_offsets, out, c_begin, c_end, iters, ring, bars);
  else
    digest_warp_ring<kPf>(n_req, offsets, tokens, chunk_offsets, pf, total, c_begin, c_end, iters, ring, bars);
}

// One warp per phase-1 range boundary b: the request holding chunks B_b - 1 and B_b, if it began
// inside range b - 1 (else an earlier boundary's warp owns it), is continued from out[B_b - 1]
// (chained by CTA b - 1) through its remaining raw digests, 32 per step: lanes load a block
// (four blocks in flight) and stage it in shared memory, every lane runs the serial chain over
// it (broadcast reads), lane k keeps value k, and the block is stored back coalesced.
constexpr int kTailWarps = 4;
__global__ void __launch_bounds__(32 * kTailWarps) k_chain_tail(int64_t n_req, const int64_t* __restrict__ co,
                                                              uint64_t* __restrict__ out, int grid) {
  __shared__ uint64_t tail_rows[kTailWarps][32];
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * kTailWarps + (threadIdx.x >> 5) + 1;
  if (b >= grid) return;
  const int64_t total = co[n_req];
  const int64_t B = total * b / grid, Bp = total * (b - 1) / grid;
  if (B >= total) return;
  const int64_t r = warp_upper_bound(co, n_req + 1, B) - 1;  // co[r] <= B < co[r + 1]
  const int64_t r0 = co[r], end = co[r + 1];
  if (r0 >= B || r0 < Bp) return;
  uint64_t* rowb = tail_rows[threadIdx.x >> 5];
  uint64_t h = out[B - 1];
  constexpr int kAhead = 4;
  uint64_t buf[kAhead];
#pragma unroll
  for (int a = 0; a < kAhead; ++a) {
    const int64_t c = B + a * 32 + lane;
    buf[a] = c < end ? out[c] : 0;
  }
  for (int64_t base = B; base < end; base += 32 * kAhead) {
#pragma unroll
    for (int a = 0; a < kAhead; ++a) {
      const int64_t blk = base + a * 32;
      if (blk < end) {
        rowb[lane] = buf[a];
        const int64_t nx = blk + 32 * kAhead + lane;
        buf[a] = nx < end ? out[nx] : 0;
        const int n = static_cast<int>(min(end - blk, int64_t{32}));
        __syncwarp();
        uint64_t mine = 0;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const uint64_t g = fpair(h, rowb[k]);
          h = k < n ? g : h;
          mine = lane == k ? g : mine;
        }
        __syncwarp();
        if (lane < n) out[blk + lane] = mine;
      }
    }
  }
}

// Phase 2 -- the per-request chain H_c = pair(H_{c-1}, digest_c), in place.  The chain is
// serial per request, so each lane owns one request; but its digests move through shared
// memory transposed, so every global access is coalesced: a round covers kSpan digests of each
// request, and one load instruction reads two requests' kSpan-digest rows (half-warp each, 128 B)
// instead of 32 scattered 8-byte words.  Round t+1's rows are loaded into registers while round t
// is folded (software pipeline).  kSpan = 16 keeps the kernel under 80 registers, so the 100K-
// request grid is a single wave and the warp holding the longest request starts at once.
// A warp runs as many rounds as its longest request, so a CTA first ranks its kChainGroup
// requests by chunk count (longest first) and hands warp w the requests of ranks [32w, 32w + 32):
// on the LooGLE 100K queue this cuts the warp-rounds from 2.36x to 1.25x the useful rounds.
constexpr int kChainWarps = 8;
constexpr int kChainGroup = 32 * kChainWarps;
constexpr int kSpan = 16;

__global__ void __launch_bounds__(kChainGroup) k_chain(
    int64_t n_req, const int64_t* __restrict__ chunk_offsets, uint64_t* __restrict__ out) {
  // [request][digest]; rows padded to 18 words: 16-byte aligned for the lane-row reads, and 8
  // consecutive rows start on distinct bank quads
  __shared__ __align__(16) uint64_t buf[kChainWarps][32][kSpan + 2];
  __shared__ int64_t sb[kChainWarps][32], sn[kChainWarps][32];
  __shared__ int64_t key[kChainGroup];
  __shared__ int16_t by_rank[kChainGroup];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int half = lane >> 4, j = lane & 15;
  const int64_t g0 = static_cast<int64_t>(blockIdx.x) * kChainGroup;
  {  // rank this CTA's requests: longer first, ties in request order (a stable sort)
    const int t = threadIdx.x;
    const int64_t mine = g0 + t < n_req ? chunk_offsets[g0 + t + 1] - chunk_offsets[g0 + t] : -1;
    key[t] = mine;
    __syncthreads();
    int rank = 0;
#pragma unroll 8
    for (int u = 0; u < kChainGroup; ++u) {
      const int64_t k = key[u];
      rank += (k > mine) | ((k == mine) & (u < t));
    }
    by_rank[rank] = static_cast<int16_t>(t);
    __syncthreads();
  }
  const int64_t r = g0 + by_rank[threadIdx.x];
  const int64_t b = r < n_req ? chunk_offsets[r] : 0;
  const int64_t n = r < n_req ? chunk_offsets[r + 1] - b : 0;
  sb[w][lane] = b;
  sn[w][lane] = n;
  const int rounds = __reduce_max_sync(0xffffffffu, static_cast<unsigned>((n + kSpan - 1) / kSpan));
  __syncwarp();
  if (rounds == 0) return;
  uint64_t (*bw)[kSpan + 2] = buf[w];
  uint64_t nx[16];  // nx[p]: digest j of request 2p+half in the next round
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    const int q = 2 * p + half;
    nx[p] = j < sn[w][q] ? out[sb[w][q] + j] : 0;
  }
  uint64_t h = (kFnvOffset << 32) | (kFnvOffset >> 32);
  for (int t = 0; t < rounds; ++t) {
    const int64_t o = static_cast<int64_t>(t) * kSpan + j;
#pragma unroll
    for (int p = 0; p < 16; ++p) bw[2 * p + half][j] = nx[p];
    __syncwarp();
    if (t + 1 < rounds) {
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        const int q = 2 * p + half;
        nx[p] = o + kSpan < sn[w][q] ? out[sb[w][q] + o + kSpan] : 0;
      }
    }
    // This lane's digests left in the round.  All shared-memory reads (128-bit) issue before the
    // serial fold, and the fold is branch-free (select), so each step costs only the two
    // dependent 64-bit FNV multiplies.
    const int m = static_cast<int>(min(n - static_cast<int64_t>(t) * kSpan, int64_t{kSpan}));
    ulonglong2 v[kSpan / 2];
#pragma unroll
    for (int k = 0; k < kSpan / 2; ++k) v[k] = reinterpret_cast<const ulonglong2*>(bw[lane])[k];
#pragma unroll
    for (int k = 0; k < kSpan / 2; ++k) {
      const uint64_t g0 = fpair(h, v[k].x);
      h = 2 * k < m ? g0 : h;
      v[k].x = h;
      const uint64_t g1 = fpair(h, v[k].y);
      h = 2 * k + 1 < m ? g1 : h;
      v[k].y = h;
    }
#pragma unroll
    for (int k = 0; k < kSpan / 2; ++k) reinterpret_cast<ulonglong2*>(bw[lane])[k] = v[k];
    __syncwarp();
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      const int q = 2 * p + half;
      if (o < sn[w][q]) out[sb[w][q] + o] = bw[q][j];
    }
    __syncwarp();
  }
}

__global__ void k_gen_tokens(uint64_t seed, const int64_t* __restrict__ offsets,
                             const int64_t* __restrict__ doc, const int64_t* __restrict__ shared_len,
                             int32_t* __restrict__ out) {
  const int64_t r = blockIdx.x;
  const int64_t t0 = offsets[r], n = offsets[r + 1] - t0;
  const int64_t sl = shared_len[r];
  const uint64_t own = (1ull << 40) + static_cast<uint64_t>(r);
  const uint64_t d = static_cast<uint64_t>(doc[r]);
  for (int64_t p = threadIdx.x; p < n; p += blockDim.x) {
    const uint64_t stream = p < sl ? d : own;
    out[t0 + p] = static_cast<int32_t>(
        mix64(seed + stream * 0x9e3779b97f4a7c15ull + static_cast<uint64_t>(p) * 0xd1b54a32d192ed03ull) >>
        47);
  }
}

}  // namespace

// Phase-1 CTAs per SM (3 shipped; tsb_hash_set_grid for measurement).  L2 prefetch one warp
// group ahead is shipped: +2.5-4% on phase 1 over both layouts, deeper prefetch loses
// (profiles/r02_k3_prefetch_sweep.jsonl).  The fused chain is a measured variant, no faster.
static int g_digest_ctas_per_sm = 3;
static int g_digest_prefetch = 1;
void set_hash_grid(int ctas_per_sm) { g_digest_ctas_per_sm = ctas_per_sm > 0 ? ctas_per_sm : 3; }
void set_hash_prefetch(int groups) { g_digest_prefetch = groups > 0 ? groups : 0; }

static int g_fused_chain = 0;
void set_hash_fused(int on) { g_fused_chain = on; }

static void launch_digest(int64_t n_req, const int64_t* offsets, const int32_t* tokens,
                          const int64_t* chunk_offsets, uint64_t* out, cudaStream_t st) {
  const int grid = 148 * g_digest_ctas_per_sm;
  if (g_digest_prefetch > 0)
    k_chunk_digest<true><<<grid, kHashThreads, 0, st>>>(n_req, offsets, tokens, chunk_offsets, out, g_digest_prefetch);
  else
    k_chunk_digest<false><<<grid, kHashThreads, 0, st>>>(n_req, offsets, tokens, chunk_offsets, out, 0);
  count_launch();
}

static void launch_fused(int64_t n_req, const int64_t* offsets, const int32_t* tokens,
                         const int64_t* chunk_offsets, uint64_t* out, cudaStream_t st) {
  const int grid = 148 * g_digest_ctas_per_sm;
  if (g_digest_prefetch > 0)
    k_chunk_hash_fused<true><<<grid, kFusedThreads, 0, st>>>(n_req, offsets, tokens, chunk_offsets, out,
                                                             g_digest_prefetch);
  else
    k_chunk_hash_fused<false><<<grid, kFusedThreads, 0, st>>>(n_req, offsets, tokens, chunk_offsets, out, 0);
  count_launch();
  k_chain_tail<<<ceil_div(grid, kTailWarps), 32 * kTailWarps, 0, st>>>(n_req, chunk_offsets, out, grid);
  count_launch();
}

cudaError_t launch_chunk_digests(int64_t n_req, const int64_t* offsets, const int32_t* tokens,
                                 const int64_t* chunk_offsets, uint64_t* out, cudaStream_t st) {
  if (n_req == 0) return cudaSuccess;
  launch_digest(n_req, offsets, tokens, chunk_offsets, out, st);
  return cudaGetLastError();
}

cudaError_t launch_hash_prefix(int64_t n_req, const int64_t* offsets, const int32_t* tokens,
                               const int64_t* chunk_offsets, uint64_t* out, cudaStream_t st) {
  if (n_req == 0) return cudaSuccess;
  // persistent phase-1 grid: 3 CTAs of 8 warps per SM (4 measured no faster)
  if (g_fused_chain) {
    launch_fused(n_req, offsets, tokens, chunk_offsets, out, st);
  } else {
    launch_digest(n_req, offsets, tokens, chunk_offsets, out, st);
    k_chain<<<ceil_div(n_req, kChainGroup), kChainGroup, 0, st>>>(n_req, chunk_offsets, out);
    count_launch();
  }
  return cudaGetLastError();
}

cudaError_t launch_gen_tokens(uint64_t seed, int64_t n_req, const int64_t* offsets,
                              const int64_t* doc, const int64_t* shared_len, int32_t* out,
                              cudaStream_t st) {
  if (n_req == 0) return cudaSuccess;
  k_gen_tokens<<<static_cast<unsigned>(n_req), 256, 0, st>>>(seed, offsets, doc, shared_len, out);
  count_launch();
  return cudaGetLastError();
}

}  // namespace tsb
