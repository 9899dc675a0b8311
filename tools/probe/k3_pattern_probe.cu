// K3 phase-1 access pattern without the request bookkeeping: is the gap to the 7.41 TB/s
// read ceiling the FNV compute or the access pattern?  1 KiB chunks, CTA-contiguous ranges,
// warps interleaved in 4-chunk groups, half-warp per chunk, two-round rotating pipeline (the
// shipped K3 structure).  MODE 0: FNV fold + 4-level shuffle tree (as K3); 1: xor-fold only;
// 2: loads only (xor of the raw words).  Probe only; not product code.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e = (x);                                                                      \
    if (e != cudaSuccess) {                                                                   \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));               \
      exit(1);                                                                                \
    }                                                                                         \
  } while (0)

constexpr uint64_t kOff = 0xcbf29ce484222325ull, kPrime = 0x100000001b3ull;
__device__ __forceinline__ uint64_t fstep(uint64_t h, uint64_t w) { return (h ^ w) * kPrime; }
__device__ __forceinline__ int4 ld(const int4* p) {
  int4 r;
  asm volatile(
      "{\n.reg .b64 pol;\ncreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], pol;\n}"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}
__device__ __forceinline__ uint64_t w64(int a, int b) {
  return static_cast<uint64_t>(static_cast<uint32_t>(a)) | (static_cast<uint64_t>(static_cast<uint32_t>(b)) << 32);
}

template <int MODE>
__device__ __forceinline__ uint64_t fold(const int4 (&v)[4]) {
  uint64_t h = kOff;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (MODE == 0) {
      h = fstep(h, w64(v[k].x, v[k].y));
      h = fstep(h, w64(v[k].z, v[k].w));
    } else {
      h ^= w64(v[k].x, v[k].y) ^ w64(v[k].z, v[k].w);
    }
  }
  return h;
}

template <int MODE>
__global__ void __launch_bounds__(256, 3) k(const int32_t* __restrict__ tok, int64_t total, uint64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31, half = lane >> 4, j = lane & 15, w = threadIdx.x >> 5;
  const int64_t c_begin = total * blockIdx.x / gridDim.x, c_end = total * (blockIdx.x + 1) / gridDim.x;
  const int64_t first = c_begin + 4 * w;
  constexpr int64_t kStride = 32;
  int4 f[2][4];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int64_t cc = first + 2 * u + half;
    if (cc < c_end)
#pragma unroll
      for (int q = 0; q < 4; ++q) f[u][q] = ld(reinterpret_cast<const int4*>(tok + cc * 256 + 64 * q + 4 * j));
  }
  uint64_t acc = 0;
  for (int64_t c = first; c < c_end; c += kStride) {
    uint64_t v[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      v[u] = fold<MODE>(f[u]);
      const int64_t nc = c + 2 * u + half + kStride;
      if (nc < c_end)
#pragma unroll
        for (int q = 0; q < 4; ++q) f[u][q] = ld(reinterpret_cast<const int4*>(tok + nc * 256 + 64 * q + 4 * j));
    }
    if (MODE == 0) {
      const uint64_t r = __shfl_xor_sync(0xffffffffu, (j & 1) ? v[0] : v[1], 1, 16);
      uint64_t x = (j & 1) ? fstep(fstep(kOff, r), v[1]) : fstep(fstep(kOff, v[0]), r);
#pragma unroll
      for (int d = 2; d < 16; d <<= 1) {
        const uint64_t o = __shfl_down_sync(0xffffffffu, x, d, 16);
        if ((j & (2 * d - 1)) < 2) x = fstep(fstep(kOff, x), o);
      }
      const int64_t cc = c + 2 * j + half;
      if (j < 2 && cc < c_end) out[cc] = x;
    } else {
      acc ^= v[0] ^ v[1];
    }
  }
  if (MODE != 0 && acc == 0x123456789ull) out[0] = acc;
}

template <class F>
float best_ms(F&& f) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 7; ++r) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, ms);
  }
  return best;
}

int main() {
  const int64_t chunks = 10922090;  // the configs[4] queue's chunk count
  int32_t* tok;
  uint64_t* out;
  CK(cudaMalloc(&tok, chunks * 1024));
  CK(cudaMalloc(&out, chunks * 8));
  CK(cudaMemset(tok, 7, chunks * 1024));
  const double bytes = chunks * 1032.0;
  for (int cps : {3, 4}) {
    const int grid = 148 * cps;
    printf("{\"cps\": %d, \"mode\": \"fnv+tree\", \"TBps\": %.3f}\n", cps,
           bytes / (best_ms([&] { k<0><<<grid, 256>>>(tok, chunks, out); }) * 1e-3) / 1e12);
    printf("{\"cps\": %d, \"mode\": \"xor-fold\", \"TBps\": %.3f}\n", cps,
           bytes / (best_ms([&] { k<1><<<grid, 256>>>(tok, chunks, out); }) * 1e-3) / 1e12);
    printf("{\"cps\": %d, \"mode\": \"loads\", \"TBps\": %.3f}\n", cps,
           bytes / (best_ms([&] { k<2><<<grid, 256>>>(tok, chunks, out); }) * 1e-3) / 1e12);
  }
  return 0;
}
