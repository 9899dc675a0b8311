// Read-only HBM bandwidth probe (streaming 16-byte loads, xor-reduced): the ceiling for K3's
// phase 1, which reads token ids once and writes 1/128 of that.  Probe only; not product code.
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

__device__ __forceinline__ int4 ld_nc(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int U>
__global__ void __launch_bounds__(256) k_read(const int4* __restrict__ src, size_t n16, int* out) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  int acc = 0;
  size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_nc(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n16; i += stride) {
    const int4 v = ld_nc(src + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x7fffffff) out[0] = acc;
}

// Warp-contiguous: each warp reads a contiguous 64 KiB span per step (K3's per-chunk pattern).
template <int U>
__global__ void __launch_bounds__(256) k_read_span(const int4* __restrict__ src, size_t n16, int* out) {
  const int lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x) >> 5;
  const size_t nw = (static_cast<size_t>(gridDim.x) * blockDim.x) >> 5;
  int acc = 0;
  for (size_t s = warp * 32 * U; s + 32 * U <= n16; s += nw * 32 * U) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_nc(src + s + u * 32 + lane);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x7fffffff) out[0] = acc;
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
  const size_t bytes = 8ull << 30, n16 = bytes / 16;
  int4* src;
  int* out;
  CK(cudaMalloc(&src, bytes));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(src, 1, bytes));
  for (int ctas_per_sm : {2, 4, 8}) {
    const int grid = 148 * ctas_per_sm;
    printf("{\"kernel\": \"strided\", \"U\": 4, \"grid\": %d, \"GBps\": %.1f}\n", grid,
           bytes / (best_ms([&] { k_read<4><<<grid, 256>>>(src, n16, out); }) * 1e-3) / 1e9);
    printf("{\"kernel\": \"strided\", \"U\": 8, \"grid\": %d, \"GBps\": %.1f}\n", grid,
           bytes / (best_ms([&] { k_read<8><<<grid, 256>>>(src, n16, out); }) * 1e-3) / 1e9);
    printf("{\"kernel\": \"span\", \"U\": 8, \"grid\": %d, \"GBps\": %.1f}\n", grid,
           bytes / (best_ms([&] { k_read_span<8><<<grid, 256>>>(src, n16, out); }) * 1e-3) / 1e9);
    printf("{\"kernel\": \"span\", \"U\": 16, \"grid\": %d, \"GBps\": %.1f}\n", grid,
           bytes / (best_ms([&] { k_read_span<16><<<grid, 256>>>(src, n16, out); }) * 1e-3) / 1e9);
  }
  int4* dst;
  CK(cudaMalloc(&dst, bytes / 2));
  printf("{\"kernel\": \"cudaMemcpy d2d 4 GiB\", \"GBps_rw\": %.1f}\n",
         bytes / (best_ms([&] { CK(cudaMemcpyAsync(dst, src, bytes / 2, cudaMemcpyDeviceToDevice)); }) * 1e-3) / 1e9);
  fflush(stdout);
  return 0;
}
