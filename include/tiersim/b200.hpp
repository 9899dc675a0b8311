// tiersim/b200.hpp — the B200 data plane behind the reference API: L2 chunk pool, L1 paged
// allocator + block_table, L2->L1 ingest, the real-time load stage and the prefix hasher.
// RAII wrappers over include/tsb_capi.h; every failure rethrows the reference exception class.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <vector>

#include "tiersim/cost_model.hpp"
#include "tiersim/events.hpp"
#include "tiersim/scheduler.hpp"
#include "tiersim/types.hpp"

namespace tiersim {

/// KV geometry of one model on one rank (KV-head shard tp_rank of tp_size).
struct KvShape {
  std::int64_t layers = 32, kv_heads = 8, head_dim = 128, dtype_bytes = 2;
  std::int64_t chunk_tokens = 256, page_tokens = 16, tp_size = 1, tp_rank = 0;
  tsb_kv_shape c_abi() const {
    return {layers, kv_heads, head_dim, dtype_bytes, chunk_tokens, page_tokens, tp_size, tp_rank};
  }
};

/// L2 tier: pinned, portable, mapped host memory; slot s holds one chunk [L][2][C][H][D].
class ChunkPool {
 public:
  ChunkPool(const KvShape& shape, std::int64_t slots) {
    const tsb_kv_shape s = shape.c_abi();
    tsb_pool* p = nullptr;
    check(tsb_pool_create(&s, slots, &p));
    p_.reset(p);
  }
  /// Peer-HBM tier: the same slot layout in `device`'s memory (read locally or over NVLink).
  static ChunkPool on_device(int device, const KvShape& shape, std::int64_t slots) {
    const tsb_kv_shape s = shape.c_abi();
    tsb_pool* p = nullptr;
    check(tsb_pool_create_device(device, &s, slots, &p));
    return ChunkPool(p);
  }
  /// Maps a pool another process exported with ipc_handle() (64 bytes).
  static ChunkPool open_ipc(const KvShape& shape, const void* handle, int owner_device,
                            std::int64_t slots) {
    const tsb_kv_shape s = shape.c_abi();
    tsb_pool* p = nullptr;
    check(tsb_pool_open_ipc(&s, handle, owner_device, slots, &p));
    return ChunkPool(p);
  }
  void ipc_handle(void* out64) const { check(tsb_pool_ipc_handle(p_.get(), out64)); }
  bool on_device() const { return tsb_pool_location_of(p_.get()) == TSB_POOL_DEVICE; }
  void* slot(std::int64_t s) { return tsb_pool_slot_ptr(p_.get(), s); }
  std::int64_t slots() const { return tsb_pool_slots(p_.get()); }
  std::int64_t chunk_bytes() const { return tsb_pool_chunk_bytes(p_.get()); }
  tsb_pool* handle() { return p_.get(); }

 private:
  explicit ChunkPool(tsb_pool* p) { p_.reset(p); }
  struct Del {
    void operator()(tsb_pool* p) const { tsb_pool_destroy(p); }
  };
  std::unique_ptr<tsb_pool, Del> p_;
};

/// L1 tier: paged HBM with TierLedger semantics (capacity = pages x page bytes).
class PagedAllocator {
 public:
  /// layout: the consumer's page layout (tsb_kv_layout: flash-attn, FlashInfer NHD or HND).
  PagedAllocator(int device, const KvShape& shape, std::int64_t num_pages, std::int64_t max_rows,
                 std::int64_t max_chunks, void* arena = nullptr, int layout = TSB_LAYOUT_FLASH_ATTN) {
    const tsb_kv_shape s = shape.c_abi();
    tsb_l1* l = nullptr;
    check(tsb_l1_create(device, &s, num_pages, max_rows, max_chunks, arena, &l));
    l_.reset(l);
    if (layout != TSB_LAYOUT_FLASH_ATTN) check(tsb_l1_set_layout(l, layout));
  }
  int layout() const { return tsb_l1_layout(l_.get()); }
  /// TierLedger::request semantics; returns Granted/Deferred and the request's block_table row.
  std::pair<bool, std::int32_t> request(std::int64_t request_id, std::int32_t block_index,
                                        std::int64_t bytes) {
    int granted = 0;
    int32_t row = -1;
    check(tsb_l1_request(l_.get(), request_id, block_index, bytes, &granted, &row));
    return {granted != 0, row};
  }
  /// Frees every page of a request; returns the deferred reservations granted by it (FIFO).
  std::vector<tsb_grant> release_request(std::int64_t request_id) {
    std::vector<tsb_grant> g(static_cast<std::size_t>(tsb_l1_deferred(l_.get())) + 1);
    int64_t n = 0;
    check(tsb_l1_release_request(l_.get(), request_id, g.data(), static_cast<int64_t>(g.size()), &n));
    g.resize(static_cast<std::size_t>(n));
    return g;
  }
  void sync_block_table(void* stream) { check(tsb_l1_sync_block_table(l_.get(), stream)); }
  std::int64_t capacity() const { return tsb_l1_capacity(l_.get()); }
  std::int64_t reserved() const { return tsb_l1_reserved(l_.get()); }
  std::int64_t page_bytes() const { return tsb_l1_page_bytes(l_.get()); }
  /// Cap on one copy-engine staging group (0: half of the ring; the load stage applies 128 MiB
  /// while a prefill shares the GPU unless a cap is set here).
  void set_ce_group_bytes(std::int64_t bytes) { check(tsb_l1_set_ce_group_bytes(l_.get(), bytes)); }
  std::int64_t ce_group_bytes() const { return tsb_l1_ce_group_bytes(l_.get()); }
  void* layer(std::int64_t l) { return tsb_l1_layer_ptr(l_.get(), l); }
  const int32_t* block_table() const { return tsb_l1_block_table_host(l_.get()); }
  tsb_l1* handle() { return l_.get(); }

 private:
  struct Del {
    void operator()(tsb_l1* l) const { tsb_l1_destroy(l); }
  };
  std::unique_ptr<tsb_l1, Del> l_;
};

/// One pcie_dispatch with real bytes: every (item, layer) of the batch, per-layer fences.
inline void ingest(PagedAllocator& l1, ChunkPool& pool, std::span<const tsb_ingest_item> items,
                   std::int64_t layer_lo, std::int64_t layer_hi, void* stream,
                   void* const* layer_events = nullptr, int mode = TSB_INGEST_AUTO) {
  check(tsb_ingest(l1.handle(), pool.handle(), items.data(), static_cast<int64_t>(items.size()),
                   layer_lo, layer_hi, mode, stream, layer_events));
}

/// Two-tier pcie_dispatch: items with src_slot < 0 come from slot ~src_slot of `tier` (HBM).
inline void ingest_tiered(PagedAllocator& l1, ChunkPool& pool, ChunkPool* tier,
                          std::span<const tsb_ingest_item> items, std::int64_t layer_lo,
                          std::int64_t layer_hi, void* stream, void* const* layer_events = nullptr,
                          int mode = TSB_INGEST_AUTO) {
  check(tsb_ingest_tiered(l1.handle(), pool.handle(), tier ? tier->handle() : nullptr, items.data(),
                          static_cast<int64_t>(items.size()), layer_lo, layer_hi, mode, stream,
                          layer_events));
}

/// The real-time load stage (SimEngine's dispatch semantics with real bytes).
class LoadStage {
 public:
  LoadStage(PagedAllocator& l1, ChunkPool& pool) {
    tsb_stage* s = nullptr;
    check(tsb_stage_create(l1.handle(), pool.handle(), &s));
    s_.reset(s);
  }
  struct Result {
    std::vector<tsb_stage_request> requests;
    tsb_stage_stats stats{};
  };
  /// HBM tier (this GPU's or a peer's device pool): a slot s < 0 names slot ~s of it.
  void set_hbm_tier(ChunkPool* tier) { check(tsb_stage_set_hbm_tier(s_.get(), tier ? tier->handle() : nullptr)); }
  /// Online mode: blocks start in an L3 host store and make the network hop L3 -> L2 for real into
  /// this stage's pool, under TierLedger(L2) + a slot free list (engine.cpp:341-364, 405-425).
  void set_l3(ChunkPool* l3, int copy_threads = 4) {
    check(tsb_stage_set_l3(s_.get(), l3 ? l3->handle() : nullptr, copy_threads));
  }
  /// A real prefill consumer: hook(user, q_index, bt_row, layer, stream) enqueues one layer after
  /// the stage made `stream` wait for that layer's fence (called from the stage's enqueue thread).
  void set_prefill_hook(tsb_prefill_hook hook, void* user) { check(tsb_stage_set_prefill_hook(s_.get(), hook, user)); }
  void set_compute_stream(void* stream) { check(tsb_stage_set_compute_stream(s_.get(), stream)); }
  /// slots[i][c] = pool slot of request i's planned chunk c (< 0: slot ~s of the HBM tier).
  /// Real-time replay of arrivals with SimEngine's control loop under config.control_mode /
  /// allocation_mode (tsb_stage_run_online).
  Result run_online(std::span<const RequestSpec> batch, const std::vector<std::vector<int64_t>>& slots,
                    const ClusterConfig& config, const CostModelPair& models, tsb_stage_options opt,
                    void* stream = nullptr) {
    return run_impl(tsb_stage_run_online, batch, slots, config, models, opt, stream);
  }
  Result run(std::span<const RequestSpec> batch, const std::vector<std::vector<int64_t>>& slots,
             const ClusterConfig& config, const CostModelPair& models, tsb_stage_options opt,
             void* stream = nullptr) {
    return run_impl(tsb_stage_run, batch, slots, config, models, opt, stream);
  }
  /// TraceEvent rows of the last run (opt.record_trace), in seq order: host-clock times for
  /// arrivals, grants, dispatches and compute completions; CUDA-event times for TransferDone.
  std::vector<TraceEvent> trace() const {
    int64_t n = 0;
    check(tsb_stage_trace(s_.get(), nullptr, 0, &n));
    std::vector<tsb_trace_row> rows(static_cast<std::size_t>(n));
    check(tsb_stage_trace(s_.get(), rows.data(), n, &n));
    std::vector<TraceEvent> out;
    out.reserve(rows.size());
    for (const auto& r : rows) out.push_back(trace_event_of(r));
    return out;
  }

 private:
  template <typename Fn>
  Result run_impl(Fn fn, std::span<const RequestSpec> batch,
                  const std::vector<std::vector<int64_t>>& slots, const ClusterConfig& config,
                  const CostModelPair& models, tsb_stage_options opt, void* stream) {
    QueueSoA q(batch, nullptr);
    std::vector<int64_t> off(1, 0), flat;
    for (const auto& s : slots) {
      flat.insert(flat.end(), s.begin(), s.end());
      off.push_back(static_cast<int64_t>(flat.size()));
    }
    double m[4];
    models.c_abi(m);
    const tsb_cluster c = config.c_abi();
    Result r;
    r.requests.resize(batch.size());
    check(fn(s_.get(), q.size(), q.get(), &c, m, off.data(), flat.data(), &opt, stream,
             r.requests.data(), &r.stats));
    return r;
  }

  struct Del {
    void operator()(tsb_stage* s) const { tsb_stage_destroy(s); }
  };
  std::unique_ptr<tsb_stage, Del> s_;
};

/// Chained 256-token prefix-chunk hashes for a batch of token sequences (K3).
inline std::vector<std::uint64_t> hash_prefix_chunks(std::span<const std::int64_t> offsets,
                                                     std::span<const std::int32_t> tokens,
                                                     void* stream = nullptr) {
  std::int64_t total = 0;
  for (std::size_t r = 0; r + 1 < offsets.size(); ++r) total += (offsets[r + 1] - offsets[r]) / 256;
  std::vector<std::uint64_t> out(static_cast<std::size_t>(total));
  std::int64_t n = 0;
  check(tsb_hash_prefix_chunks(stream, static_cast<int64_t>(offsets.size()) - 1, offsets.data(),
                               tokens.data(), out.data(), &n));
  return out;
}

}  // namespace tiersim
