// verify.cu — harness check of ingested pages at full size, independent of the ingest kernels.
//
// The ingest kernels map a source position to a page (seg_addr in ingest.cu).  This check walks
// the other way: it starts from the DESTINATION -- a page id of the arena, inverted on the host
// from the block table into (pool slot, first token of the page in its chunk) -- and derives, for
// every 8-byte word of the page, the (layer, K|V, token, head, dim word) it must hold from the
// consumer's layout definition alone, then the word's source index in the chunk layout
// [L][2][C][H][D] (north_star).  It shares no address arithmetic with ingest.cu:
// only the raw shape, the layout enum and the synthetic generator (synth_word) are common.
#include "common.cuh"
#include "kernels.h"

namespace tsb {
namespace {

__global__ void k_verify_pages(PageCheck c, const uint8_t* __restrict__ arena,
                               const PageSource* __restrict__ pages, int64_t n_pages,
                               uint64_t seed, unsigned long long* mismatches) {
  const int64_t dw = c.D * c.E / 8;           // 8-byte words per head row
  const int64_t plane_w = c.P * c.Hl * dw;    // words of one (layer, K|V, page) plane
  const int64_t plane_b = plane_w * 8;
  const int64_t n_layers = c.layer_hi - c.layer_lo;
  const int64_t units = n_pages * n_layers * 2;
  unsigned long long bad = 0;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t p = u / (n_layers * 2);
    const int64_t l = c.layer_lo + (u / 2) % n_layers;
    const int64_t kv = u & 1;
    const PageSource ps = pages[p];
    // destination plane of (layer l, K|V, page) in the consumer's layout
    const int64_t layer_base = l * 2 * c.num_pages * plane_b;
    const int64_t plane = c.layout == TSB_LAYOUT_FLASH_ATTN
                              ? layer_base + (kv * c.num_pages + ps.page) * plane_b
                              : layer_base + (static_cast<int64_t>(ps.page) * 2 + kv) * plane_b;
    const uint64_t* dst = reinterpret_cast<const uint64_t*>(arena + plane);
    const uint64_t chunk_w0 = static_cast<uint64_t>(ps.slot) * (c.pool_chunk_bytes / 8);
    for (int64_t w = threadIdx.x; w < plane_w; w += blockDim.x) {
      int64_t t, h;
      const int64_t x = w % dw;
      if (c.layout == TSB_LAYOUT_FLASHINFER_HND) {  // [Hl][P][D]
        h = w / (c.P * dw);
        t = (w / dw) % c.P;
      } else {  // [P][Hl][D]
        t = w / (c.Hl * dw);
        h = (w / dw) % c.Hl;
      }
      // chunk [L][2][C][H][D]: token tok0 + t, global head tp_rank * Hl + h
      const int64_t src_w = (((l * 2 + kv) * c.C + ps.tok0 + t) * c.H + c.tp_rank * c.Hl + h) * dw + x;
      bad += dst[w] != synth_word(seed, chunk_w0 + static_cast<uint64_t>(src_w));
    }
  }
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(mismatches, bad);
}

}  // namespace

cudaError_t launch_verify_pages(const PageCheck& c, const uint8_t* arena, const PageSource* pages,
                                int64_t n_pages, uint64_t seed, unsigned long long* mismatches,
                                cudaStream_t st) {
  if (n_pages == 0 || c.layer_hi <= c.layer_lo) return cudaSuccess;
  k_verify_pages<<<148 * 8, 256, 0, st>>>(c, arena, pages, n_pages, seed, mismatches);
  count_launch();
  return cudaGetLastError();
}

}  // namespace tsb
