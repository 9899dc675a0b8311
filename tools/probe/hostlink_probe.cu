// Host-link microbenchmark: copy-engine H2D vs SM zero-copy loads vs bulk-async
// (cp.async.bulk) reads of mapped pinned host memory. Probe only; not product code.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ int4 ld_nc(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ int4 ld_nc256(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ld_nc128(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::128B.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// warp-contiguous variant: each warp copies a contiguous 32 KiB span (like an ingest segment)
template <int U, int HINT>
__global__ void zc_seg(const int4* __restrict__ src, int4* __restrict__ dst, size_t nseg) {
  const int lane = threadIdx.x & 31;
  size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t s = warp; s < nseg; s += nw) {
    const int4* sp = src + s * 2048; int4* dp = dst + s * 2048;
    for (int v0 = lane; v0 < 2048; v0 += 32 * U) {
      int4 b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) b[u] = HINT == 256 ? ld_nc256(sp + v0 + u * 32) : HINT == 128 ? ld_nc128(sp + v0 + u * 32) : ld_nc(sp + v0 + u * 32);
#pragma unroll
      for (int u = 0; u < U; ++u) dp[v0 + u * 32] = b[u];
    }
  }
}

template <int U>
__global__ void zc_copy(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = tid;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_nc(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n16; i += stride) dst[i] = ld_nc(src + i);
}

// Bulk-async: one elected thread per CTA streams segments through a smem ring.
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" :: "r"(a), "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* g, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(g), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(g), "r"((uint32_t)__cvta_generic_to_shared(smem)), "r"(bytes) : "memory");
}

template <int STAGES, int SEG>
__global__ void bulk_copy(const char* __restrict__ src, char* __restrict__ dst, size_t nseg) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t bars[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;");
  size_t first = blockIdx.x, step = gridDim.x;
  // prologue
  int issued = 0;
  size_t seg = first;
  for (int s = 0; s < STAGES && seg < nseg; ++s, seg += step, ++issued) {
    mbar_expect(&bars[s], SEG);
    bulk_g2s(smem + s * SEG, src + seg * SEG, SEG, &bars[s]);
  }
  size_t cons = first;
  int k = 0;
  for (; cons < nseg; cons += step, ++k) {
    int s = k % STAGES;
    uint32_t ph = (k / STAGES) & 1;
    mbar_wait(&bars[s], ph);
    bulk_s2g(dst + cons * SEG, smem + s * SEG, SEG);
    asm volatile("cp.async.bulk.commit_group;");
    if (seg < nseg) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      mbar_expect(&bars[s], SEG);
      bulk_g2s(smem + s * SEG, src + seg * SEG, SEG, &bars[s]);
      seg += step;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  size_t bytes = (argc > 1 ? atoll(argv[1]) : 4096ll) << 20;
  char* h;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  for (size_t i = 0; i < bytes; i += 4096) h[i] = (char)i;
  char* hd;
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  char* d;
  CK(cudaMalloc(&d, bytes));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto best = [&](auto fn, int reps) {
    float bestms = 1e30f;
    for (int r = 0; r < reps; ++r) {
      CK(cudaEventRecord(a));
      fn();
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      bestms = std::min(bestms, ms);
    }
    CK(cudaGetLastError());
    return bytes / (bestms * 1e-3) / 1e9;
  };
  printf("{\"bytes\": %zu}\n", bytes);
  printf("CE_H2D GB/s %.2f\n", best([&] { CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice)); }, 5));
  printf("CE_D2H GB/s %.2f\n", best([&] { CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost)); }, 3));
  for (int g : {32, 64, 148}) {
    printf("ZCSEG nohint grid %d GB/s %.2f\n", g, best([&] { zc_seg<8, 0><<<g, 256>>>((const int4*)hd, (int4*)d, bytes / 32768); }, 3));
    printf("ZCSEG L2::128B grid %d GB/s %.2f\n", g, best([&] { zc_seg<8, 128><<<g, 256>>>((const int4*)hd, (int4*)d, bytes / 32768); }, 3));
    printf("ZCSEG L2::256B grid %d GB/s %.2f\n", g, best([&] { zc_seg<8, 256><<<g, 256>>>((const int4*)hd, (int4*)d, bytes / 32768); }, 3));
  }
  int grids[] = {64};
  for (int g : grids) {
    for (int t : {256, 512}) {
      double gbs = best([&] { zc_copy<8><<<g, t>>>((const int4*)hd, (int4*)d, bytes / 16); }, 3);
      printf("ZC_LDG128 grid %d threads %d U8 GB/s %.2f\n", g, t, gbs);
    }
  }
  {
    constexpr int ST = 4, SEG = 32768;
    CK(cudaFuncSetAttribute(bulk_copy<ST, SEG>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * SEG));
    for (int g : {8, 16, 32, 64, 148}) {
      double gbs = best([&] { bulk_copy<ST, SEG><<<g, 32, ST * SEG>>>(hd, d, bytes / SEG); }, 3);
      printf("BULK 4x32K grid %d GB/s %.2f\n", g, gbs);
    }
  }
  {
    constexpr int ST = 6, SEG = 32768;
    CK(cudaFuncSetAttribute(bulk_copy<ST, SEG>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * SEG));
    for (int g : {16, 32, 64, 148}) {
      double gbs = best([&] { bulk_copy<ST, SEG><<<g, 32, ST * SEG>>>(hd, d, bytes / SEG); }, 3);
      printf("BULK 6x32K grid %d GB/s %.2f\n", g, gbs);
    }
  }
  {
    constexpr int ST = 8, SEG = 4096;
    CK(cudaFuncSetAttribute(bulk_copy<ST, SEG>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * SEG));
    for (int g : {32, 64, 148, 296}) {
      double gbs = best([&] { bulk_copy<ST, SEG><<<g, 32, ST * SEG>>>(hd, d, bytes / SEG); }, 3);
      printf("BULK 8x4K grid %d GB/s %.2f\n", g, gbs);
    }
  }
  // verify last copy
  std::vector<char> chk(1 << 20);
  CK(cudaMemcpy(chk.data(), d + bytes - (1 << 20), 1 << 20, cudaMemcpyDeviceToHost));
  size_t bad = 0;
  for (size_t i = 0; i < (1u << 20); i += 4096) bad += chk[i] != h[bytes - (1 << 20) + i];
  printf("verify_bad %zu\n", bad);
  return 0;
}
