// Host-link concurrency probe: does the copy engine leave link bandwidth unused that SM
// zero-copy loads can take at the same time?  One process, one context.  A fraction f of the
// bytes goes by cudaMemcpyAsync (copy engine) on one stream while a zero-copy kernel (16-byte
// ld.global.nc from mapped pinned memory, G CTAs) moves the rest on another; aggregate GB/s =
// all bytes / (first start .. last end).  Also: two processes give 58.6 GB/s together where one
// copy engine gives 55.6 (bench.py --gpus 2 under TSB_BENCH_ONE_DEVICE=1).  Probe only.
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

// warp-contiguous 32 KiB spans, 8 loads in flight per lane (the K1 pattern)
__global__ void __launch_bounds__(256) zc(const int4* __restrict__ src, int4* __restrict__ dst, size_t nseg) {
  const int lane = threadIdx.x & 31;
  size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t s = warp; s < nseg; s += nw) {
    const int4* sp = src + s * 2048;
    int4* dp = dst + s * 2048;
    for (int v0 = lane; v0 < 2048; v0 += 256) {
      int4 b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) b[u] = ld_nc(sp + v0 + u * 32);
#pragma unroll
      for (int u = 0; u < 8; ++u) dp[v0 + u * 32] = b[u];
    }
  }
}

int main(int argc, char** argv) {
  const size_t total = (argc > 1 ? atoll(argv[1]) : 4096ull) << 20;
  uint8_t *h, *d, *hdev;
  CK(cudaHostAlloc(&h, total, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hdev), h, 0));
  CK(cudaMalloc(&d, total));
  for (size_t i = 0; i < total; i += 4096) h[i] = static_cast<uint8_t>(i >> 12);
  cudaStream_t sa, sb;
  CK(cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
  cudaEvent_t e0, ea, eb;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&ea));
  CK(cudaEventCreate(&eb));
  const size_t seg = 32768;
  for (int grid : {16, 32, 64}) {
    for (double f : {1.0, 0.95, 0.9, 0.85, 0.8, 0.7, 0.0}) {
      const size_t ce = (static_cast<size_t>(total * f) / seg) * seg;
      const size_t zb = total - ce;
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        CK(cudaEventRecord(e0, sa));
        CK(cudaStreamWaitEvent(sb, e0, 0));
        if (ce) CK(cudaMemcpyAsync(d, h, ce, cudaMemcpyHostToDevice, sa));
        if (zb)
          zc<<<grid, 256, 0, sb>>>(reinterpret_cast<const int4*>(hdev + ce), reinterpret_cast<int4*>(d + ce),
                                   zb / seg);
        CK(cudaEventRecord(ea, sa));
        CK(cudaEventRecord(eb, sb));
        CK(cudaEventSynchronize(ea));
        CK(cudaEventSynchronize(eb));
        float ma, mb;
        CK(cudaEventElapsedTime(&ma, e0, ea));
        CK(cudaEventElapsedTime(&mb, e0, eb));
        if (rep) best = std::min(best, std::max(ma, mb));
      }
      printf("{\"zc_grid\": %d, \"ce_frac\": %.2f, \"GBps\": %.2f}\n", grid, f, total / (best * 1e-3) / 1e9);
      fflush(stdout);
      if (f == 1.0 && grid != 16) continue;
    }
  }
  // two copy-engine streams, halves of the buffer
  for (int k : {2, 4}) {
    cudaStream_t ss[4];
    for (int i = 0; i < k; ++i) CK(cudaStreamCreateWithFlags(&ss[i], cudaStreamNonBlocking));
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0, ss[0]));
      for (int i = 1; i < k; ++i) CK(cudaStreamWaitEvent(ss[i], e0, 0));
      for (int i = 0; i < k; ++i)
        CK(cudaMemcpyAsync(d + i * (total / k), h + i * (total / k), total / k, cudaMemcpyHostToDevice, ss[i]));
      for (int i = 1; i < k; ++i) {
        CK(cudaEventRecord(ea, ss[i]));
        CK(cudaStreamWaitEvent(ss[0], ea, 0));
      }
      CK(cudaEventRecord(eb, ss[0]));
      CK(cudaEventSynchronize(eb));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, eb));
      if (rep) best = std::min(best, ms);
    }
    printf("{\"ce_streams\": %d, \"GBps\": %.2f}\n", k, total / (best * 1e-3) / 1e9);
  }
  return 0;
}
