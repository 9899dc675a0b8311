// prefill.cu — K6 synthetic prefill (benchmark harness only).
//
// Stands in for the prefill compute the reference models as
// compute_base + compute_per_token * n (+ quadratic) seconds (engine.cpp:210-212, types.hpp:90-92)
// so ingest/prefill overlap can be measured (config 4).  Each launch occupies `ctas` CTAs of 256
// threads that spin on %globaltimer for `ns` nanoseconds; the stage splits a request's prefill into
// per-layer launches of at most ~250 us so a higher-priority ingest stream can interleave its
// scatter kernels between them, as it would between real prefill kernels.
#include "common.cuh"
#include "kernels.h"

namespace tsb {
namespace {

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256) k_prefill_burn(uint64_t ns, unsigned long long* sink) {
  const uint64_t t0 = globaltimer();
  uint64_t x = threadIdx.x + 1, it = 0;
  while (globaltimer() - t0 < ns) {
#pragma unroll 8
    for (int k = 0; k < 64; ++k) x = x * 6364136223846793005ull + 1442695040888963407ull;
    ++it;
  }
  if (x == 0 && sink) atomicAdd(sink, it);  // never true; keeps the loop alive
}

}  // namespace

cudaError_t launch_prefill_burn(uint64_t ns, int ctas, unsigned long long* sink, cudaStream_t st) {
  if (ns == 0) return cudaSuccess;
  k_prefill_burn<<<ctas, 256, 0, st>>>(ns, sink);
  count_launch();
  return cudaGetLastError();
}

}  // namespace tsb
