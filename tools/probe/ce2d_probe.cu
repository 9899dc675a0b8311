// Copy-engine probe for head-sharded chunks: can the copy engines pull a rank's KV-head slice
// (runs of `w` bytes at a 2 KiB stride) from pinned host memory at the contiguous H2D rate?
// Compares one contiguous cudaMemcpyAsync, one cudaMemcpy2DAsync of the whole slice, and one
// cudaMemcpy2DAsync per (chunk, layer) = 512 rows (K and V of 256 tokens).  (The r01 run also
// timed the batched 3D-copy entry point; it is closed on this pool since, so the variant is gone.)
// Probe only; not product code.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e = (x);                                                                      \
    if (e != cudaSuccess) {                                                                   \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));               \
      exit(1);                                                                                \
    }                                                                                         \
  } while (0)

template <class F>
double best_gbps(size_t payload, cudaStream_t st, F&& f, int reps = 5) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaStreamSynchronize(st));
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a, st));
    f();
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, ms);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return payload / (best * 1e-3) / 1e9;
}

int main(int argc, char** argv) {
  const size_t payload = (argc > 1 ? atoll(argv[1]) : 1024) << 20;  // bytes moved per test
  const size_t row = 2048;                                            // H*D*E at 8 heads
  const size_t host_bytes = payload * (row / 256);                    // enough for w=256
  uint8_t *h = nullptr, *d = nullptr;
  CK(cudaHostAlloc(&h, host_bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  CK(cudaMalloc(&d, payload));
  for (size_t i = 0; i < host_bytes; i += 4096) h[i] = static_cast<uint8_t>(i >> 12);
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));

  printf("{\"test\": \"contig\", \"GBps\": %.2f}\n",
         best_gbps(payload, st, [&] { CK(cudaMemcpyAsync(d, h, payload, cudaMemcpyHostToDevice, st)); }));

  for (size_t w : {256, 512, 1024, 2048}) {
    const size_t height = payload / w;
    printf("{\"test\": \"2d_single\", \"w\": %zu, \"GBps\": %.2f}\n", w,
           best_gbps(payload, st, [&] {
             CK(cudaMemcpy2DAsync(d, w, h, row, w, height, cudaMemcpyHostToDevice, st));
           }));
    const size_t rows_per_op = 512;  // one (chunk, layer): K and V of 256 tokens
    const size_t nops = payload / (w * rows_per_op);
    // One cudaMemcpy2DAsync per (chunk, layer) op (per-call overhead).
    printf("{\"test\": \"2d_per_op\", \"w\": %zu, \"ops\": %zu, \"GBps\": %.2f}\n", w, nops,
           best_gbps(payload, st, [&] {
             for (size_t k = 0; k < nops; ++k)
               CK(cudaMemcpy2DAsync(d + k * rows_per_op * w, w, h + k * rows_per_op * row, row, w,
                                    rows_per_op, cudaMemcpyHostToDevice, st));
           }, 3));
  }
  // One 3D op per (layer, run of consecutive slots): width w, height 512 rows at pitch `row`,
  // depth = run slots at a slice pitch of one chunk (L * 512 rows).  L = 80 (Llama-3-70B).
  const size_t L = 80, chunk_rows = L * 512;
  for (size_t w : {256, 512, 1024}) {
    const size_t slice = 512 * w;  // one item's layer slice, packed
    const size_t n_items = payload / slice;
    const size_t chunk_bytes = chunk_rows * row;
    const size_t slots_fit = host_bytes / chunk_bytes;
    for (size_t run : {size_t(1), size_t(4), size_t(16), size_t(64), size_t(100)}) {
      if (run > slots_fit) continue;
      const size_t nops = n_items / run;
      auto go = [&] {
        for (size_t k = 0; k < nops; ++k) {
          cudaMemcpy3DParms p = {};
          const size_t slot0 = (k * run) % (slots_fit - run + 1);
          p.srcPtr = make_cudaPitchedPtr(h + slot0 * chunk_bytes + (k % L) * 512 * row, row, w, chunk_rows);
          p.dstPtr = make_cudaPitchedPtr(d + k * run * slice, w, w, 512);
          p.extent = make_cudaExtent(w, 512, run);
          p.kind = cudaMemcpyHostToDevice;
          CK(cudaMemcpy3DAsync(&p, st));
        }
      };
      printf("{\"test\": \"3d_run\", \"w\": %zu, \"run\": %zu, \"ops\": %zu, \"GBps\": %.2f}\n", w, run,
             nops, best_gbps(nops * run * slice, st, go, 3));
    }
  }
  fflush(stdout);
  return 0;
}
