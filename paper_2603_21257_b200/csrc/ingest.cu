// ingest.cu — K1 (zero-copy / bulk) and K2 (staged scatter) ingest kernels for sm_100a.
//
// The L2->L1 hop the reference only models as `transfer_base_latency + bytes/pcie_bandwidth`
// per chunk (engine.cpp:206-207), dispatched one chunk at a time by pcie_dispatch
// (engine.cpp:427-446).  Here one launch moves a batch of chunks x a layer range.  Work unit:
// a segment = (item, layer, K|V, page j) = page_tokens rows of `run` bytes gathered from the
// chunk [L][2][C][H][D] and written contiguously into page block_table[row][chunk*ppc + j]
// of the layer's [2][num_pages][P][H_local][D] arena.  Segments are numbered so consecutive
// ids read consecutive source bytes (layer-major inside a chunk), which keeps host reads
// sequential.  No tensor cores: a pure gather/scatter bounded by the host link (K1) or HBM (K2).
#include <cuda.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace tsb {
namespace {

struct SegAddr {
  const uint8_t* src;
  uint8_t* dst;
  bool ok;
};

__device__ __forceinline__ SegAddr seg_addr(const IngestGeom& g, const uint8_t* src,
                                            uint8_t* arena, const tsb_ingest_item* items,
                                            const int32_t* bt, int64_t s) {
  const int64_t spi = static_cast<int64_t>(g.n_layers) * 2 * g.ppc;
  const int64_t i = s / spi;
  const int64_t r = s - i * spi;
  const int64_t l = r / (2 * g.ppc);
  const int64_t kv = (r / g.ppc) & 1;
  const int64_t j = r % g.ppc;
  const tsb_ingest_item it = items[i];
  const int32_t page = bt[static_cast<int64_t>(it.bt_row) * g.bt_stride +
                          static_cast<int64_t>(it.chunk_index) * g.ppc + j];
  SegAddr a;
  const int64_t base = g.staged ? i * g.item_stride
                                : it.src_slot * g.chunk_bytes + g.layer_lo * g.layer_src;
  a.src = src + base + l * g.layer_src + kv * g.kv_src + j * g.P * g.row + g.head_off;
  a.dst = arena + (g.layer_lo + l) * g.layer_dst + kv * g.kv_dst +
          static_cast<int64_t>(page) * g.page_dst;
  a.ok = page >= 0 && page < g.num_pages;
  return a;
}

// K1 / K2: one warp per segment, 16-byte streaming loads, U loads in flight per lane before
// the stores.  Source may be mapped host memory (K1, zero-copy over PCIe) or an HBM staging
// buffer (K2).  NHD pages keep the source order.  HND pages ([H_local][P][D]) are walked in
// destination order: the stores are contiguous and the loads gather each head's row of token t
// (walking in source order with transposed stores measured 0.93 of HBM at TP2/TP4 vs 0.95-0.96,
// repo:profiles/r02_k1_hnd_walk.jsonl).
__device__ __forceinline__ int64_t hnd_src_off(const IngestGeom& g, int v, int vph) {
  // destination order [h][t][w] -> source [t][h][w] (32-bit index math)
  const int per_head = static_cast<int>(g.P) * vph;
  const int h = v / per_head, rem = v - h * per_head;
  const int t = rem / vph, w = rem - t * vph;
  return static_cast<int64_t>(t) * g.row + static_cast<int64_t>(h) * g.head_bytes + w * 16;
}

template <bool kContig, int U, bool kHnd>
__global__ void __launch_bounds__(256) k_ingest_ldg(IngestGeom g, const uint8_t* __restrict__ src,
                                                    uint8_t* __restrict__ arena,
                                                    const tsb_ingest_item* __restrict__ items,
                                                    const int32_t* __restrict__ bt,
                                                    int64_t nseg) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int vpr = static_cast<int>(g.run >> 4);
  const int vph = static_cast<int>(g.head_bytes >> 4);
  const int nvec = static_cast<int>(g.P) * vpr;
  for (int64_t s = warp; s < nseg; s += nwarps) {
    const SegAddr a = seg_addr(g, src, arena, items, bt, s);
    if (!a.ok) continue;
    for (int v0 = lane; v0 < nvec; v0 += 32 * U) {
      int4 buf[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = v0 + u * 32;
        if (v < nvec) {
          const int64_t off = kHnd      ? hnd_src_off(g, v, vph)
                              : kContig ? static_cast<int64_t>(v) * 16
                                        : (v / vpr) * g.row + (v % vpr) * 16;
          buf[u] = ld_stream(a.src + off);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = v0 + u * 32;
        if (v < nvec) st_stream(a.dst + static_cast<int64_t>(v) * 16, buf[u]);
      }
    }
  }
}

// K1b: the TMA engine does the moving, from a tensor map.  The source is a 2D (NHD pages) or 3D
// (HND pages) tensor map over the pool -- or over the CE staging ring -- whose box is exactly one
// page segment: P token rows x this rank's run for NHD, or [H_local][P][D] for HND, where the map's
// dimension order (D, token rows, heads) makes the TMA unit perform the per-head transpose on the
// way into shared memory.  So one UTMALDG brings a whole (layer, K|V, page) segment, at any head
// shard (TP8: one 4 KiB box instead of 16 row copies), and one cp.async.bulk stores it to the page.
// One warp per CTA, lane 0 issues; a ring of `stages` segment buffers completes on mbarriers.
__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* m, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* smem, const CUtensorMap* m, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

template <bool kHnd>
__global__ void __launch_bounds__(32) k_ingest_tma(const __grid_constant__ CUtensorMap src_map, IngestGeom g,
                                                   TmaSrc ts, uint8_t* __restrict__ arena,
                                                   const tsb_ingest_item* __restrict__ items,
                                                   const int32_t* __restrict__ bt, int64_t nseg, int stages) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[kTmaMaxStages];
  // Addresses of this CTA's segments, 64 iterations in a ring: the whole warp resolves 32 of them
  // at a time (item and block-table loads in parallel), so lane 0's TMA loop never waits on a
  // dependent global load.
  __shared__ int32_t row_tab[64];
  __shared__ uint8_t* dst_tab[64];
  const int lane = threadIdx.x;
  const uint32_t seg = static_cast<uint32_t>(g.seg_bytes);
  const int64_t grid = gridDim.x;
  const int64_t spi = static_cast<int64_t>(g.n_layers) * 2 * g.ppc;
  auto resolve = [&](int64_t k) {  // iteration k of this CTA -> table slot k % 64
    const int64_t s = blockIdx.x + k * grid;
    if (s >= nseg) return;
    const int64_t i = s / spi, r = s - i * spi;
    const int64_t l = r / (2 * g.ppc), kv = (r / g.ppc) & 1, j = r % g.ppc;
    // token-row coordinate in the source map: rows are [slot][L][2][C] (pool) or
    // [item][n_layers][2][C] (staging ring)
    const int64_t outer = g.staged ? i * g.n_layers + l : items[i].src_slot * ts.layers + g.layer_lo + l;
    row_tab[k & 63] = static_cast<int32_t>((outer * 2 + kv) * ts.C + j * g.P);
    const SegAddr a = seg_addr(g, nullptr, arena, items, bt, s);
    dst_tab[k & 63] = a.ok ? a.dst : nullptr;
  };
  auto issue = [&](int64_t k) {
    const int st = static_cast<int>(k % stages);
    uint8_t* buf = smem + static_cast<int64_t>(st) * seg;
    mbar_arrive_expect_tx(&full[st], seg);
    if (kHnd)
      tma_load_3d(buf, &src_map, 0, row_tab[k & 63], ts.head0, &full[st]);
    else
      tma_load_2d(buf, &src_map, ts.x0, row_tab[k & 63], &full[st]);
  };
  if (lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&src_map)) : "memory");
    for (int st = 0; st < stages; ++st) mbar_init(&full[st], 1);
    mbar_fence_init();
  }
  resolve(lane);
  resolve(32 + lane);
  __syncwarp();
  if (lane == 0)
    for (int64_t k = 0; k < stages && blockIdx.x + k * grid < nseg; ++k) issue(k);
  // Iteration k consumes this CTA's k-th segment from stage k % stages.  A stage is refilled
  // kLag - 1 iterations after its store was committed (wait_group.read kLag-1), so up to kLag
  // stores read shared memory while the next loads are already in flight.
  constexpr int kLag = 3;
  for (int64_t k = 0; blockIdx.x + k * grid < nseg; ++k) {
    if ((k & 31) == 0 && k > 0) {  // all of this block's and the next block's entries resolved
      __syncwarp();
      resolve(k + 32 + lane);
      __syncwarp();
    }
    if (lane == 0) {
      const int st = static_cast<int>(k % stages);
      mbar_wait(&full[st], static_cast<uint32_t>((k / stages) & 1));
      uint8_t* dst = dst_tab[k & 63];
      if (dst) bulk_s2g(dst, smem + static_cast<int64_t>(st) * seg, seg);
      bulk_commit();
      const int64_t j = k - (kLag - 1);  // its store is now at most kLag-1 groups from the newest
      if (j >= 0 && blockIdx.x + (j + stages) * grid < nseg) {
        bulk_wait_read<kLag - 1>();
        issue(j + stages);
      }
    }
  }
  if (lane == 0) bulk_wait0();
}

// K8: chunk replication inside L1.  A chunk already resident in one request's pages is copied
// into another request's pages (HBM -> HBM) instead of crossing the host link again -- LooGLE-like
// batches read each document chunk from several requests.  Warp per (item, layer, K|V, page)
// plane; both sides use the arena's layout, so a plane is one contiguous seg_bytes copy.
__global__ void __launch_bounds__(256) k_page_copy(IngestGeom g, uint8_t* __restrict__ arena,
                                                   const tsb_page_copy* __restrict__ items,
                                                   const int32_t* __restrict__ bt, int64_t nseg) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t spi = static_cast<int64_t>(g.n_layers) * 2 * g.ppc;
  const int nvec = static_cast<int>(g.seg_bytes >> 4);
  for (int64_t s = warp; s < nseg; s += nwarps) {
    const int64_t i = s / spi, r = s - i * spi;
    const int64_t l = g.layer_lo + r / (2 * g.ppc), kv = (r / g.ppc) & 1, j = r % g.ppc;
    const tsb_page_copy it = items[i];
    const int32_t ps = bt[static_cast<int64_t>(it.src_row) * g.bt_stride + static_cast<int64_t>(it.src_chunk) * g.ppc + j];
    const int32_t pd = bt[static_cast<int64_t>(it.dst_row) * g.bt_stride + static_cast<int64_t>(it.dst_chunk) * g.ppc + j];
    if (ps < 0 || pd < 0 || ps >= g.num_pages || pd >= g.num_pages) continue;
    const uint8_t* src = arena + l * g.layer_dst + kv * g.kv_dst + static_cast<int64_t>(ps) * g.page_dst;
    uint8_t* dst = arena + l * g.layer_dst + kv * g.kv_dst + static_cast<int64_t>(pd) * g.page_dst;
    for (int v0 = lane; v0 < nvec; v0 += 32 * 4) {
      int4 buf[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (v0 + u * 32 < nvec) buf[u] = ld_stream(src + static_cast<int64_t>(v0 + u * 32) * 16);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (v0 + u * 32 < nvec) st_stream(dst + static_cast<int64_t>(v0 + u * 32) * 16, buf[u]);
    }
  }
}

__global__ void k_fill_synth(uint64_t* __restrict__ dst, uint64_t first_word, uint64_t n_words,
                             uint64_t seed) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t npairs = n_words / 2;
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < npairs;
       p += stride) {
    const uint64_t w = first_word + 2 * p;
    const uint64_t a = synth_word(seed, w), b = synth_word(seed, w + 1);
    int4 v;
    v.x = static_cast<int>(a);
    v.y = static_cast<int>(a >> 32);
    v.z = static_cast<int>(b);
    v.w = static_cast<int>(b >> 32);
    *reinterpret_cast<int4*>(dst + 2 * p) = v;
  }
  if ((n_words & 1) && blockIdx.x == 0 && threadIdx.x == 0)
    dst[n_words - 1] = synth_word(seed, first_word + n_words - 1);
}

template <bool kHnd>
void launch_ldg_variant(const IngestGeom& g, const uint8_t* src, uint8_t* arena,
                        const tsb_ingest_item* items, const int32_t* bt, int64_t nseg, int grid,
                        cudaStream_t st, bool hbm_source) {
  const bool contig = g.run == g.row;
  if (hbm_source) {
    if (contig)
      k_ingest_ldg<true, 4, kHnd><<<grid, 256, 0, st>>>(g, src, arena, items, bt, nseg);
    else
      k_ingest_ldg<false, 4, kHnd><<<grid, 256, 0, st>>>(g, src, arena, items, bt, nseg);
  } else {
    if (contig)
      k_ingest_ldg<true, 8, kHnd><<<grid, 256, 0, st>>>(g, src, arena, items, bt, nseg);
    else
      k_ingest_ldg<false, 8, kHnd><<<grid, 256, 0, st>>>(g, src, arena, items, bt, nseg);
  }
}

}  // namespace

cudaError_t launch_ingest_ldg(const IngestGeom& g, const uint8_t* src, uint8_t* arena,
                              const tsb_ingest_item* items, const int32_t* bt, int64_t n_items,
                              int grid, cudaStream_t st, bool hbm_source) {
  const int64_t nseg = n_items * g.n_layers * 2 * g.ppc;
  if (nseg == 0) return cudaSuccess;
  // Loads in flight per lane: 8 over the host link (microsecond latency, 64 CTAs); 4 from HBM,
  // where the sweep (profiles/r01_k1_sweep.jsonl) peaks with 4 loads per lane and a 32-CTA-per-
  // SM grid: 6.54-6.63 TB/s for full-head segments (U=8: 6.06-6.10 at 1184 CTAs).
  if (g.hnd)
    launch_ldg_variant<true>(g, src, arena, items, bt, nseg, grid, st, hbm_source);
  else
    launch_ldg_variant<false>(g, src, arena, items, bt, nseg, grid, st, hbm_source);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_ingest_tma(const CUtensorMap& src_map, const IngestGeom& g, const TmaSrc& ts, uint8_t* arena,
                              const tsb_ingest_item* items, const int32_t* bt, int64_t n_items, int grid,
                              cudaStream_t st) {
  const int64_t nseg = n_items * g.n_layers * 2 * g.ppc;
  if (nseg == 0) return cudaSuccess;
  static std::atomic<uint64_t> attr_set{0};
  if (first_on_device(attr_set)) {
    cudaError_t e = cudaFuncSetAttribute(k_ingest_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBulkSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_ingest_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBulkSmem);
    if (e != cudaSuccess) return e;
  }
  // ring depth: as many segment buffers as fit (6 for 32 KiB segments, 16 for TP8's 4 KiB)
  const int stages = tma_ring_stages(g.seg_bytes);
  const size_t smem = static_cast<size_t>(stages) * g.seg_bytes;
  if (g.hnd)
    k_ingest_tma<true><<<grid, 32, smem, st>>>(src_map, g, ts, arena, items, bt, nseg, stages);
  else
    k_ingest_tma<false><<<grid, 32, smem, st>>>(src_map, g, ts, arena, items, bt, nseg, stages);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_page_copy(const IngestGeom& g, uint8_t* arena, const tsb_page_copy* items, const int32_t* bt,
                             int64_t n_items, int grid, cudaStream_t st) {
  const int64_t nseg = n_items * g.n_layers * 2 * g.ppc;
  if (nseg == 0) return cudaSuccess;
  k_page_copy<<<grid, 256, 0, st>>>(g, arena, items, bt, nseg);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_fill_synth(uint64_t* dst, uint64_t first_word, uint64_t n_words, uint64_t seed,
                              cudaStream_t st) {
  if (n_words == 0) return cudaSuccess;
  k_fill_synth<<<148 * 8, 256, 0, st>>>(dst, first_word, n_words, seed);
  count_launch();
  return cudaGetLastError();
}

}  // namespace tsb
