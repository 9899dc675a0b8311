// hash.cu — K3 warp-parallel prefix chunk hasher (+ synthetic token generator) for sm_100a.
//
// The reference's only hash is byte-serial FNV-1a-64 (engine.cpp:500-507), used for a config
// fingerprint; it has no prefix hasher.  The definition frozen in
// oracle/tsb_oracle.c (orc_hash_prefix_chunks) keeps FNV-1a's constants and step but makes a
// 256-token chunk warp-parallel: lane j folds tokens [8j, 8j+8) as 64-bit FNV words, a 5-level
// shuffle tree pairs the 32 leaves, and the chunk digests are chained per request so hash c
// names the whole prefix [0, 256(c+1)).  One warp per request, kUnroll chunks in flight.
// HBM-bound: 4 B/token read + 8 B/chunk written.
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

__device__ __forceinline__ uint64_t leaf8(const int32_t (&t)[8]) {
  uint64_t h = kFnvOffset;
#pragma unroll
  for (int k = 0; k < 8; ++k) h = fstep(h, static_cast<uint64_t>(static_cast<uint32_t>(t[k])));
  return h;
}

__device__ __forceinline__ uint64_t tree32(uint64_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t o = __shfl_down_sync(0xffffffffu, v, d);
    if ((lane & (2 * d - 1)) == 0) v = fpair(v, o);
  }
  return v;  // valid in lane 0
}

__device__ __forceinline__ void load8(const int32_t* p, bool aligned, int32_t (&t)[8]) {
  if (aligned) {
    const int4 a = __ldg(reinterpret_cast<const int4*>(p));
    const int4 b = __ldg(reinterpret_cast<const int4*>(p) + 1);
    t[0] = a.x; t[1] = a.y; t[2] = a.z; t[3] = a.w;
    t[4] = b.x; t[5] = b.y; t[6] = b.z; t[7] = b.w;
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) t[k] = __ldg(p + k);
  }
}

// One warp per request: chunks are processed kUnroll at a time (all their loads issued before
// any is consumed), lane 0 folds each digest into the request's chain as it goes and stores the
// running hash.  No block-level synchronisation; ~kUnroll KiB in flight per warp.
constexpr int kUnroll = 4;

__global__ void __launch_bounds__(kHashThreads) k_hash_prefix(int64_t n_req,
                                                              const int64_t* __restrict__ offsets,
                                                              const int32_t* __restrict__ tokens,
                                                              const int64_t* __restrict__ chunk_offsets,
                                                              uint64_t* __restrict__ out) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(kHashWarps) + (threadIdx.x >> 5);
  if (r >= n_req) return;
  const int lane = threadIdx.x & 31;
  const int64_t t0 = offsets[r];
  const int64_t nchunks = (offsets[r + 1] - t0) / 256;
  const int64_t c0 = chunk_offsets[r];
  const bool aligned = (t0 & 3) == 0;
  const int32_t* base = tokens + t0 + lane * 8;
  uint64_t h = (kFnvOffset << 32) | (kFnvOffset >> 32);
  for (int64_t c = 0; c < nchunks; c += kUnroll) {
    int32_t tk[kUnroll][8];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (c + u < nchunks) load8(base + (c + u) * 256, aligned, tk[u]);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (c + u < nchunks) {
        const uint64_t d = tree32(leaf8(tk[u]), lane);
        if (lane == 0) {
          h = fpair(h, d);
          out[c0 + c + u] = h;
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
