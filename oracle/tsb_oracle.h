/*
 * tsb_oracle.h — CPU restatement of the CALVO KV-ingest hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2603_21257_b200/, include/)
 * links, loads or calls this; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg do, and only as the checker or the CPU arm.
 *
 * Pinning: the planning, ledger, cost, key and order functions are checked bit-for-bit
 * against the reference's own sources compiled in place (oracle/_ref, see Makefile) and
 * against the golden vectors of the reference tests (tests/golden/).  The data-plane
 * functions (scatter, page allocation, prefix hash) have no counterpart in the reference
 * (SURVEY.md 8(c)); they restate the reference semantics they cite plus the north-star
 * layouts, and the byte-wise FNV-1a primitive is pinned against the reference's
 * config_fingerprint (engine.cpp:500-534).
 */
#ifndef TSB_ORACLE_H_
#define TSB_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same field order and meaning as tiersim::ClusterConfig (types.hpp:82-97). */
typedef struct {
  double network_bandwidth;
  double pcie_bandwidth;
  double transfer_base_latency;
  int64_t l1_capacity;
  int64_t l2_capacity;
  int64_t bytes_per_token;
  int64_t block_size_tokens;
  double compute_base;
  double compute_per_token;
  double compute_quadratic;
  int32_t allocation_mode; /* 0 proactive, 1 reactive */
  int32_t control_mode;    /* 0 coupled, 1 decoupled */
} orc_cluster;

/* Struct-of-arrays view of a queue of tiersim::RequestSpec (types.hpp:52-64). */
enum { ORC_HAS_DEADLINE = 1, ORC_HAS_MEASURED = 2 };
typedef struct {
  const int64_t* id;
  const double* arrival;
  const int64_t* context_tokens;
  const int64_t* query_tokens;
  const double* cache_hit_ratio;
  const uint8_t* flags;
  const double* deadline;
  const double* measured_t_load;
  const double* measured_t_comp;
} orc_queue;

/* Status codes: identical values to tsb_status in include/tsb_capi.h. */
enum {
  ORC_OK = 0,
  ORC_VALIDATION = 1,
  ORC_CAPACITY = 2,
  ORC_MISSING_DEADLINE = 3,
  ORC_DEGENERATE_FIT = 4
};

/* Policies in tiersim::PolicyKind order (scheduler.hpp:23). */
enum { ORC_FIFO = 0, ORC_SJF_PT = 1, ORC_SJF_COST = 2, ORC_EDF = 3, ORC_LSTF = 4 };

/* ---- planning arithmetic (types.cpp) ---- */
int orc_kv_bytes_per_token(int64_t layers, int64_t kv_heads, int64_t head_dim,
                           int64_t dtype_bytes, int64_t* out);
int64_t orc_cached_token_count(int64_t context_tokens, double hit, int64_t block_size);
int64_t orc_compute_token_count(int64_t context_tokens, int64_t query_tokens, double hit,
                                int64_t block_size);

/* ---- cost model (cost_model.cpp) ---- */
double orc_predict(double slope, double intercept, int64_t tokens);
void orc_cost_models_from_config(const orc_cluster* c, double out_models[4]);
int orc_fit_linear(int64_t n, const int64_t* tokens, const double* seconds, double* slope,
                   double* intercept, int* slope_clamped, int* intercept_clamped);

/* ---- batched scorer + order (cost_model.cpp:56-71, scheduler.cpp:39-100) ---- */
int orc_score_queue(int64_t n, const orc_queue* q, int policy, const double models[4],
                    const orc_cluster* c, double* t_load, double* t_comp, double* primary,
                    int64_t* err_index);
int orc_key_less(double pa, double aa, int64_t ia, double pb, double ab, int64_t ib);
int orc_sort_order(int64_t n, const double* primary, const double* arrival, const int64_t* id,
                   int64_t* order);
int orc_drain_order(int64_t n, const double* primary, const double* arrival,
                    const int64_t* id, int64_t* order);

/* ---- TierLedger (engine.cpp:18-49) ---- */
typedef struct orc_ledger orc_ledger;
orc_ledger* orc_ledger_new(int64_t capacity);
void orc_ledger_free(orc_ledger* l);
int orc_ledger_request(orc_ledger* l, int64_t request_id, int32_t block_index, int64_t bytes,
                       int* granted);
int orc_ledger_release(orc_ledger* l, int64_t bytes, int64_t* req_out, int32_t* blk_out,
                       int64_t* bytes_out, int64_t cap, int64_t* n_out);
int64_t orc_ledger_reserved(const orc_ledger* l);
int64_t orc_ledger_deferred(const orc_ledger* l);

/* ---- paged allocator restatement (alloc_ref): FIFO free list of page ids ---- */
typedef struct orc_pages orc_pages;
orc_pages* orc_pages_new(int64_t num_pages);
void orc_pages_free(orc_pages* p);
int64_t orc_pages_take(orc_pages* p, int64_t n, int32_t* out);
void orc_pages_give(orc_pages* p, int64_t n, const int32_t* ids);
int64_t orc_pages_available(const orc_pages* p);

/* ---- KV geometry ----
 * Chunk (L2, LMCache-style):   [layers][2][chunk_tokens][kv_heads][head_dim] elements
 * Paged (L1, vLLM flash-attn): per layer [2][num_pages][page_tokens][heads_local][head_dim]
 *                              stored as one arena [layers][2][num_pages][...].            */
typedef struct {
  int64_t layers, kv_heads, head_dim, dtype_bytes;
  int64_t chunk_tokens, page_tokens;
  int64_t tp_size, tp_rank;
} orc_kv_shape;

/* One (request, chunk) transfer: chunk `src_slot` of the pool lands in the pages
 * block_table[bt_row][chunk_index*pages_per_chunk + j]. */
typedef struct {
  int64_t src_slot;
  int32_t bt_row;
  int32_t chunk_index;
} orc_ingest_item;

void orc_scatter_ref(const orc_kv_shape* s, const uint8_t* pool, int64_t n_items,
                     const orc_ingest_item* items, const int32_t* block_table,
                     int64_t bt_stride, int64_t num_pages, uint8_t* arena, int64_t layer_lo,
                     int64_t layer_hi, int threads);
/* layout: 0 flash-attn [2][pages][P][Hl][D], 1 FlashInfer NHD [pages][2][P][Hl][D],
 * 2 FlashInfer HND [pages][2][Hl][P][D] (per layer). */
void orc_scatter_ref_layout(const orc_kv_shape* s, const uint8_t* pool, int64_t n_items,
                            const orc_ingest_item* items, const int32_t* block_table,
                            int64_t bt_stride, int64_t num_pages, uint8_t* arena, int64_t layer_lo,
                            int64_t layer_hi, int threads, int layout);
void orc_scatter_ref_window(const orc_kv_shape* s, const uint8_t* pool, int64_t n_items,
                            const orc_ingest_item* items, const int32_t* block_table,
                            int64_t bt_stride, int64_t num_pages, uint8_t* arena_window,
                            int64_t layer_lo, int64_t layer_hi, int threads, int layout);

/* synthetic data */
uint64_t orc_mix64(uint64_t x);
uint64_t orc_synth_word(uint64_t seed, uint64_t word_index);
void orc_synth_fill(uint64_t seed, uint64_t first_word, uint64_t n_words, uint64_t* out,
                    int threads);
uint32_t orc_token_id(uint64_t seed, uint64_t stream, uint64_t pos);
void orc_gen_tokens(uint64_t seed, int64_t n_req, const int64_t* offsets, const int64_t* doc,
                    const int64_t* shared_len, int32_t* out, int threads);

/* hashing */
uint64_t orc_fnv1a_bytes(uint64_t h, const void* data, size_t len);
uint64_t orc_chunk_digest(const int32_t* tokens256);
uint64_t orc_chain(uint64_t prev, uint64_t digest);
int64_t orc_hash_prefix_chunks(int64_t n_req, const int64_t* offsets, const int32_t* tokens,
                               const int64_t* chunk_offsets, uint64_t* out, int threads);

#ifdef __cplusplus
}
#endif
#endif
