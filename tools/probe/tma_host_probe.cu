// Probe: tensor-map TMA (cp.async.bulk.tensor, SASS UTMALDG) reading mapped pinned host memory,
// against the copy engine and the non-tensor cp.async.bulk (UBLKCP).  Question: does the TMA
// tensor path (with L2 promotion 128B/256B) issue larger PCIe read requests than the SMs' 128 B
// and so beat the 51.5 GB/s SM ceiling measured in round 1?  Probe only; not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_host_probe tma_host_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
#define CU(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, s); exit(1);} } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(sa(b)),
               "r"(ph));
}
__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* m, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          sa(smem)),
      "l"(m), "r"(x), "r"(y), "r"(sa(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(sa(smem)), "r"(bytes)
               : "memory");
}

// Tile t = rows [t*BY, t*BY+BY) x columns [x0, x0+BX) (u64 elements) of the host tensor; written
// contiguously to dst + t*tile_bytes.
template <int STAGES>
__global__ void tma_copy(const __grid_constant__ CUtensorMap src, char* __restrict__ dst, int ntiles, int x0, int by,
                         uint32_t tile_bytes) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint64_t bars[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;");
  int t_issue = blockIdx.x, k_issue = 0;
  for (; k_issue < STAGES && t_issue < ntiles; ++k_issue, t_issue += gridDim.x) {
    mbar_expect(&bars[k_issue], tile_bytes);
    tma_load_2d(smem + k_issue * tile_bytes, &src, x0, t_issue * by, &bars[k_issue]);
  }
  int k = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % STAGES;
    mbar_wait(&bars[s], (k / STAGES) & 1);
    bulk_s2g(dst + (size_t)t * tile_bytes, smem + s * tile_bytes, tile_bytes);
    asm volatile("cp.async.bulk.commit_group;");
    if (t_issue < ntiles) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      mbar_expect(&bars[s], tile_bytes);
      tma_load_2d(smem + s * tile_bytes, &src, x0, t_issue * by, &bars[s]);
      t_issue += gridDim.x;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const size_t bytes = (size_t)(argc > 1 ? atoll(argv[1]) : 4096) << 20;
  const int row_bytes = 2048;  // one token row of [H=8][D=128] bf16
  const size_t rows = bytes / row_bytes;
  char* h;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  for (size_t i = 0; i < bytes; i += 8) *(uint64_t*)(h + i) = i * 0x9E3779B97F4A7C15ull;
  char* hd;
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  char* d;
  CK(cudaMalloc(&d, bytes));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto best = [&](auto fn, size_t moved, int reps) {
    float bm = 1e30f;
    for (int r = 0; r < reps; ++r) {
      CK(cudaEventRecord(a));
      fn();
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      bm = std::min(bm, ms);
    }
    CK(cudaGetLastError());
    return moved / (bm * 1e-3) / 1e9;
  };
  printf("CE_H2D GB/s %.2f\n", best([&] { CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice)); }, bytes, 5));

  const char* pname[] = {"none", "64B", "128B", "256B"};
  CUtensorMapL2promotion promos[] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
  struct Cfg { int bx, by, x0; const char* what; };
  // bx in u64 elements: 256 = full 2 KiB row (full heads), 32 = 256 B (one TP8 head slice), 64 = TP4
  Cfg cfgs[] = {{256, 16, 0, "full-heads 2KiBx16"}, {256, 32, 0, "full-heads 2KiBx32"},
                {32, 16, 0, "tp8 256Bx16"}, {32, 128, 0, "tp8 256Bx128"}, {32, 256, 96, "tp8 256Bx256 rank3"},
                {64, 64, 0, "tp4 512Bx64"}, {128, 64, 128, "tp2 1KiBx64 rank1"}};
  for (auto& cf : cfgs) {
    for (int p = 0; p < 4; ++p) {
      CUtensorMap m;
      cuuint64_t dims[2] = {(cuuint64_t)(row_bytes / 8), (cuuint64_t)rows};
      cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
      cuuint32_t box[2] = {(cuuint32_t)cf.bx, (cuuint32_t)cf.by};
      cuuint32_t es[2] = {1, 1};
      CU(cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, hd, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promos[p],
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
      const uint32_t tile = cf.bx * 8 * cf.by;
      const int ntiles = (int)(rows / cf.by);
      const size_t moved = (size_t)ntiles * tile;
      for (int stages : {4, 8}) {
        const size_t sm = (size_t)stages * tile;
        if (sm > 200 * 1024) continue;
        for (int grid : {32, 148, 296}) {
          double g;
          if (stages == 4) {
            CK(cudaFuncSetAttribute(tma_copy<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            g = best([&] { tma_copy<4><<<grid, 32, sm>>>(m, d, ntiles, cf.x0, cf.by, tile); }, moved, 3);
          } else {
            CK(cudaFuncSetAttribute(tma_copy<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            g = best([&] { tma_copy<8><<<grid, 32, sm>>>(m, d, ntiles, cf.x0, cf.by, tile); }, moved, 3);
          }
          printf("TMA %-22s promo %-4s stages %d grid %3d GB/s %.2f\n", cf.what, pname[p], stages, grid, g);
        }
      }
      // verify the last launch: tile 1, row r, column x0.. of the source
      std::vector<uint64_t> chk(tile / 8);
      CK(cudaMemcpy(chk.data(), d + tile, tile, cudaMemcpyDeviceToHost));
      size_t bad = 0;
      for (int r = 0; r < cf.by; ++r)
        for (int x = 0; x < cf.bx; ++x)
          bad += chk[r * cf.bx + x] != *(uint64_t*)(h + (size_t)(cf.by + r) * row_bytes + (cf.x0 + x) * 8);
      printf("TMA %-22s promo %-4s verify_bad %zu\n", cf.what, pname[p], bad);
    }
  }
  return 0;
}
