// kernels.h — launch interface of the sm_100a kernels (internal to libtsb.so).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "tsb_capi.h"

namespace tsb {

// Geometry of one ingest launch.  A "segment" is one (item, layer, K|V, page) unit: P token
// rows of `run` bytes read at stride `row` from the chunk, written contiguously to one page.
struct IngestGeom {
  int64_t row;          // H*D*E: one token's K (or V) across all heads in the chunk
  int64_t run;          // H_local*D*E: this rank's slice of that row
  int64_t head_off;     // tp_rank*H_local*D*E
  int64_t chunk_bytes;  // L*2*C*row: one L2 slot
  int64_t kv_src;       // C*row: K->V stride inside a chunk layer
  int64_t layer_src;    // 2*C*row
  int64_t P;            // page tokens
  int64_t ppc;          // pages per chunk (C/P)
  int64_t seg_bytes;    // P*run
  int64_t num_pages;
  int64_t kv_dst;       // K -> V plane stride of the destination (layout-dependent)
  int64_t page_dst;     // page stride of the destination (layout-dependent)
  int64_t layer_dst;    // 2*num_pages*seg_bytes
  int64_t head_bytes;   // D*E: one head's row inside a page
  int32_t hnd;          // 1: pages are [H_local][P][D] (TSB_LAYOUT_FLASHINFER_HND), else [P][H_local][D]
  int64_t bt_stride;    // block_table row stride (int32 entries)
  int32_t layer_lo;     // first layer of the launch
  int32_t n_layers;     // layers in the launch
  // Source addressing: slot mode (src = base + slot*chunk_bytes + layer_lo*layer_src) for the
  // L2 pool, or staged mode (src = base + item_rank*item_stride) for a CE staging buffer that
  // holds only layers [layer_lo, layer_lo+n_layers) of each item.
  int32_t staged;
  int64_t item_stride;
};

// hbm_source: the source is device memory (HBM staging ring, local or peer HBM pool) rather
// than mapped host memory; picks the loads-in-flight depth.
cudaError_t launch_ingest_ldg(const IngestGeom& g, const uint8_t* src, uint8_t* arena,
                              const tsb_ingest_item* items, const int32_t* bt, int64_t n_items,
                              int grid, cudaStream_t st, bool hbm_source);
// K1b: one tensor-map TMA load per page segment (ingest.cu).  TmaSrc carries what the map's
// coordinates need beyond IngestGeom: the pool's layer count and chunk tokens (rows are
// [slot][L][2][C]) and this rank's first head (HND maps) or first u64 column (NHD maps).
constexpr int kBulkSmem = 200 * 1024;
constexpr int kTmaMaxStages = 16;
// Ring depth per CTA: ~96 KiB of segments (6..16 stages, within kBulkSmem), ~64 KiB for head-
// shard segments of <= 8 KiB so three rings share an SM (TP4's 8 KiB segments: 0.876 -> 0.902
// of HBM, TP8 unchanged; repo:profiles/r02_k1b_ring_sweep.jsonl).  Full-head 32 KiB segments run
// one 6-deep ring per SM.
inline int tma_ring_stages(int64_t seg_bytes) {
  int64_t st = (seg_bytes <= 8192 ? 65536 : 98304) / seg_bytes;
  st = st < 6 ? 6 : st > kTmaMaxStages ? kTmaMaxStages : st;
  while (st > 2 && st * seg_bytes > kBulkSmem) --st;
  return static_cast<int>(st);
}
inline int tma_ctas_per_sm(int64_t seg_bytes) {
  const int64_t ring = tma_ring_stages(seg_bytes) * seg_bytes + 2048;
  const int64_t n = (228 * 1024) / ring;
  return static_cast<int>(n < 1 ? 1 : n > 4 ? 4 : n);
}
struct TmaSrc {
  int64_t layers;  // L of the source chunks (slot mode)
  int64_t C;       // chunk tokens
  int32_t x0;      // NHD map: first 8-byte column of this rank's run in a token row
  int32_t head0;   // HND map: first head of this rank
};
cudaError_t launch_ingest_tma(const CUtensorMap& src_map, const IngestGeom& g, const TmaSrc& ts, uint8_t* arena,
                              const tsb_ingest_item* items, const int32_t* bt, int64_t n_items, int grid,
                              cudaStream_t st);
// K8: copy resident chunks' pages to other rows' pages (HBM -> HBM), layers of g.
cudaError_t launch_page_copy(const IngestGeom& g, uint8_t* arena, const tsb_page_copy* items, const int32_t* bt,
                             int64_t n_items, int grid, cudaStream_t st);
cudaError_t launch_fill_synth(uint64_t* dst, uint64_t first_word, uint64_t n_words, uint64_t seed,
                              cudaStream_t st);
// Harness page check (verify.cu): the canonical shape and layout only, no IngestGeom.
struct PageCheck {
  int64_t H, Hl, D, E, C, P, tp_rank;  // chunk [L][2][C][H][D]; this rank's heads [tp_rank*Hl, +Hl)
  int64_t num_pages;
  int64_t pool_chunk_bytes;  // slot stride of the pool whose synthetic pattern is expected
  int32_t layout;            // tsb_kv_layout
  int32_t layer_lo, layer_hi;
};
struct PageSource {  // inverted block table: which chunk position a page must hold
  int64_t slot;      // pool slot of the chunk
  int32_t page;      // page id in the arena
  int32_t tok0;      // first token of the page inside the chunk (j * P)
};
cudaError_t launch_verify_pages(const PageCheck& c, const uint8_t* arena, const PageSource* pages,
                                int64_t n_pages, uint64_t seed, unsigned long long* mismatches,
                                cudaStream_t st);

// Scorer (K4) and order (K5).
struct ScoreParams {
  int policy;
  double load_slope, load_icpt, comp_slope, comp_icpt;
  double quadratic;
  int64_t block;
};
cudaError_t launch_score(int64_t n, tsb_queue q, ScoreParams p, double* t_load, double* t_comp,
                         double* primary, uint64_t* kp, uint64_t* ka, uint64_t* ki,
                         unsigned long long* err_missing, unsigned long long* err_nan,
                         cudaStream_t st);
// Sorts (kp, ka, ki) ascending, producing the permutation in order_out.  Scratch must hold
// 2 * n of each key array plus 2 * n int64 indices.  *sorted (device) must be nonzero on entry;
// it is cleared when the keys are not already in order (then the merge sort runs).
cudaError_t launch_order(int64_t n, uint64_t* kp, uint64_t* ka, uint64_t* ki, int64_t* idx,
                         uint64_t* kp2, uint64_t* ka2, uint64_t* ki2, int64_t* idx2,
                         int64_t* order_out, unsigned long long* sorted, cudaStream_t st);

// Prefix hasher (K3) and token generator.
void set_hash_grid(int ctas_per_sm);
void set_hash_prefetch(int groups);
void set_hash_fused(int on);
cudaError_t launch_chunk_digests(int64_t n_req, const int64_t* offsets, const int32_t* tokens,
                                 const int64_t* chunk_offsets, uint64_t* out, cudaStream_t st);
cudaError_t launch_hash_prefix(int64_t n_req, const int64_t* offsets, const int32_t* tokens,
                               const int64_t* chunk_offsets, uint64_t* out, cudaStream_t st);
cudaError_t launch_gen_tokens(uint64_t seed, int64_t n_req, const int64_t* offsets,
                              const int64_t* doc, const int64_t* shared_len, int32_t* out,
                              cudaStream_t st);

// L2 chunk index (K7).
cudaError_t launch_index_insert(uint64_t* keys, int64_t* vals, uint64_t* owner, uint64_t mask,
                                int64_t n, const uint64_t* hashes, const int64_t* slots,
                                uint64_t epoch, int64_t* pos, unsigned long long* stats,
                                cudaStream_t st);
cudaError_t launch_index_rehash(const uint64_t* okeys, const int64_t* ovals, const uint64_t* oowner,
                                uint64_t cap, uint64_t* keys, int64_t* vals, uint64_t* owner,
                                uint64_t mask, cudaStream_t st);
cudaError_t launch_index_erase(uint64_t* keys, uint64_t mask, int64_t n, const uint64_t* hashes,
                               unsigned long long* stats, cudaStream_t st);
cudaError_t launch_index_lookup(const uint64_t* keys, const int64_t* vals, uint64_t mask,
                                int64_t n_req, const int64_t* chunk_offsets,
                                const uint64_t* hashes, int64_t* slots_out, int64_t* matched,
                                cudaStream_t st);

// Synthetic prefill burner (K6, harness).
cudaError_t launch_prefill_burn(uint64_t ns, int ctas, unsigned long long* sink, cudaStream_t st);

}  // namespace tsb
