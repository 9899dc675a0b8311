// hash.cu — K3 warp-parallel prefix chunk hasher (+ synthetic token generator) for sm_100a.
//
// The reference's only hash is byte-serial FNV-1a-64 (engine.cpp:500-507), used for a config
// fingerprint; it has no prefix hasher.  The definition frozen in
// oracle/tsb_oracle.c (orc_hash_prefix_chunks) keeps FNV-1a's constants and step, applied to
// 64-bit words (two int32 token ids each): 16 leaves of 8 words per 256-token chunk, a 4-level
// pairwise tree, and a per-request chain so hash c names the whole prefix [0, 256(c+1)).
//
// Mapping: one warp per request; each half-warp owns one chunk per round (lane j of the half
// folds leaf j = words 32k+2j, 32k+2j+1 for k = 0..3, so each of the four 16-byte load
// instructions reads 2 x 256 contiguous bytes -- fully coalesced), two rounds are loaded before any
// is consumed (4 chunks = 4 KiB in flight per warp), the tree is 4 shuffle levels inside the
// half-warp, and lane 0 folds both digests into the chain.  HBM-bound: 4 B/token + 8 B/chunk.
#include "common.cuh"
#include "kernels.h"

namespace tsb {
namespace {

__device__ __forceinline__ uint64_t fstep(uint64_t h, uint64_t w) { return (h ^ w) * kFnvPrime; }
__device__ __forceinline__ uint64_t fpair(uint64_t a, uint64_t b) {
  return fstep(fstep(kFnvOffset, a), b);
}

constexpr int kHashThreads = 256;
constexpr int kHashWarps = kHashThreads / 32;
constexpr int kRounds = 2;  // rounds of 2 chunks loaded ahead per warp

struct Leaf {
  int4 v[4];  // 16 int32 tokens
};

// Lane j of a half-warp loads tokens [64k + 4j, 64k + 4j + 4) for k = 0..3: every 16-byte load
// instruction of the warp reads two contiguous 256-byte runs (one per chunk).
__device__ __forceinline__ void load_leaf(const int32_t* p, bool aligned, Leaf& f) {
  if (aligned) {
#pragma unroll
    for (int k = 0; k < 4; ++k) f.v[k] = ld_stream(p + 64 * k);
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

// 4-level pairwise tree over the 16 leaves of each half-warp; result in lanes 0 and 16.
__device__ __forceinline__ uint64_t tree16(uint64_t v, int j) {
#pragma unroll
  for (int d = 1; d < 16; d <<= 1) {
    const uint64_t o = __shfl_down_sync(0xffffffffu, v, d, 16);
    if ((j & (2 * d - 1)) == 0) v = fpair(v, o);
  }
  return v;
}

__global__ void __launch_bounds__(kHashThreads, 4) k_hash_prefix(
    int64_t n_req, const int64_t* __restrict__ offsets, const int32_t* __restrict__ tokens,
    const int64_t* __restrict__ chunk_offsets, uint64_t* __restrict__ out) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(kHashWarps) + (threadIdx.x >> 5);
  if (r >= n_req) return;
  const int lane = threadIdx.x & 31;
  const int half = lane >> 4, j = lane & 15;
  const int64_t t0 = offsets[r];
  const int64_t nchunks = (offsets[r + 1] - t0) / 256;
  uint64_t* dst = out + chunk_offsets[r];
  const bool aligned = (t0 & 3) == 0;
  const int32_t* base = tokens + t0 + half * 256 + j * 4;
  uint64_t h = (kFnvOffset << 32) | (kFnvOffset >> 32);
  for (int64_t c = 0; c < nchunks; c += 2 * kRounds) {
    Leaf f[kRounds];
#pragma unroll
    for (int u = 0; u < kRounds; ++u)
      if (c + 2 * u + half < nchunks) load_leaf(base + (c + 2 * u) * 256, aligned, f[u]);
#pragma unroll
    for (int u = 0; u < kRounds; ++u) {
      const int64_t ca = c + 2 * u;
      if (ca >= nchunks) break;
      const uint64_t d = tree16(fold_leaf(f[u]), j);
      const uint64_t db = __shfl_sync(0xffffffffu, d, 16);
      if (lane == 0) {
        h = fpair(h, d);
        dst[ca] = h;
        if (ca + 1 < nchunks) {
          h = fpair(h, db);
          dst[ca + 1] = h;
        }
      }
    }
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

cudaError_t launch_hash_prefix(int64_t n_req, const int64_t* offsets, const int32_t* tokens,
                               const int64_t* chunk_offsets, uint64_t* out, cudaStream_t st) {
  if (n_req == 0) return cudaSuccess;
  const int64_t grid = (n_req + kHashWarps - 1) / kHashWarps;
  k_hash_prefix<<<static_cast<unsigned>(grid), kHashThreads, 0, st>>>(n_req, offsets, tokens,
                                                                     chunk_offsets, out);
  count_launch();
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
