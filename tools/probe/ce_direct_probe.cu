// Probe: can the copy engines scatter chunks straight into pages (no K2, no SMs)?
// One cudaMemcpyAsync per (layer, K|V, page run) segment -- 32 KiB contiguous on both sides per
// page for full-head chunks -- to randomly permuted page destinations, 32 KiB (fully fragmented
// pages) to 1 MiB (a chunk's 16 pages on consecutive ids, K and V).  Also under a concurrent
// SM-saturating kernel (stand-in for prefill) to show the copy engines are unaffected.
// (r02 first ran this with the batched-memcpy entry point, since closed on this pool.)
// Probe only; not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ce_direct_probe ce_direct_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void burn(float* out, int iters) {  // keeps every SM busy (FMA chain per thread)
  float a = threadIdx.x * 1e-3f, b = 1.0001f;
  for (int i = 0; i < iters; ++i) a = fmaf(a, b, 1e-7f);
  if (a == 12345.f) out[0] = a;
}

int main(int argc, char** argv) {
  const size_t bytes = (size_t)(argc > 1 ? atoll(argv[1]) : 4096) << 20;
  char* h;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  for (size_t i = 0; i < bytes; i += 4096) h[i] = (char)(i >> 12);
  char* d;
  CK(cudaMalloc(&d, bytes));
  float* sink;
  CK(cudaMalloc(&sink, 4));
  cudaStream_t s, sb;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  std::mt19937_64 rng(1);
  for (size_t seg : {size_t(32) << 10, size_t(64) << 10, size_t(256) << 10, size_t(1) << 20}) {
    const size_t n = bytes / seg;
    std::vector<size_t> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    std::shuffle(perm.begin(), perm.end(), rng);
    std::vector<void*> dst(n), src(n);
    for (size_t i = 0; i < n; ++i) {
      src[i] = h + i * seg;
      dst[i] = d + perm[i] * seg;
    }
    for (int busy = 0; busy < 2; ++busy) {
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        if (busy) burn<<<148 * 8, 256, 0, sb>>>(sink, 1 << 22);  // ~tens of ms of full-GPU FMA
        CK(cudaEventRecord(a, s));
        for (size_t i = 0; i < n; ++i) CK(cudaMemcpyAsync(dst[i], src[i], seg, cudaMemcpyHostToDevice, s));
        CK(cudaEventRecord(b, s));
        CK(cudaEventSynchronize(b));
        CK(cudaStreamSynchronize(sb));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        best = std::min(best, ms);
      }
      printf("{\"probe\": \"ce_percall_scatter\", \"segment_bytes\": %zu, \"entries\": %zu, \"sm_busy\": %d, "
             "\"GBps\": %.2f}\n", seg, n, busy, bytes / (best * 1e-3) / 1e9);
    }
  }
  // verify one permutation sample of the last configuration (1 MiB segments)
  std::vector<char> chk(4096);
  CK(cudaMemcpy(chk.data(), d, 4096, cudaMemcpyDeviceToHost));
  printf("{\"verify_first_byte\": %d}\n", (int)chk[0]);
  return 0;
}
