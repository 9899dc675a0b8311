/*
 * tsb_capi.h — C ABI of the B200-native CALVO KV-ingest path (libtsb.so).
 *
 * Plain pointers and sizes only; no torch or C++ types cross this boundary.  Every entry
 * point returns a tsb_status; on failure tsb_last_error() (thread-local) holds the message,
 * worded like the reference's throw sites so the C++ shim (include/tiersim/ headers) and the
 * Python mirror can rethrow the matching error.hpp class.
 *
 * Each declaration cites the reference interface it replaces (paths relative to
 * /root/reference/proj/).  The reference has no device or process boundary (SURVEY.md 0,
 * 8(b)); the L2->L1 hop it models in engine.cpp:206-207 / :427-446 is the one this ABI
 * makes real.
 *
 * Threading: one host thread per device issues calls; device work is asynchronous on the
 * caller's stream (a cudaStream_t passed as void*, NULL = legacy default stream) unless the
 * function says it synchronises.  Objects are not thread-safe (like TierLedger,
 * engine.hpp:48-52).
 */
#ifndef TSB_CAPI_H_
#define TSB_CAPI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  Mapping to reference exceptions (core/include/tiersim/error.hpp:13-71). */
typedef enum {
  TSB_OK = 0,
  TSB_VALIDATION = 1,       /* ValidationError */
  TSB_CAPACITY = 2,         /* CapacityError */
  TSB_MISSING_DEADLINE = 3, /* MissingDeadline */
  TSB_DEGENERATE_FIT = 4,   /* DegenerateFit */
  TSB_CUDA = 5,             /* CUDA runtime failure (tiersim::Error) */
  TSB_UNSUPPORTED = 6,      /* shape/option not supported by the kernels */
  TSB_UNKNOWN_PROFILE = 7   /* UnknownProfile (builtin_profile, workload.cpp:35) */
} tsb_status;

const char* tsb_last_error(void);
const char* tsb_version(void);
/* The calling thread's current CUDA device (cudaGetDevice; 0 if none), for header-only C++
 * callers that keep one object per device. */
int tsb_current_device(void);
/* Number of device kernels this library has launched since load (evidence counter). */
uint64_t tsb_kernel_launch_count(void);

/* ------------------------------------------------------------------------------------ */
/* Cluster calibration: field-for-field tiersim::ClusterConfig (types.hpp:82-97).          */
/* ------------------------------------------------------------------------------------ */
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
  int32_t allocation_mode; /* 0 Proactive, 1 Reactive (types.hpp:70) */
  int32_t control_mode;    /* 0 Coupled, 1 Decoupled (types.hpp:71) */
} tsb_cluster;

/* Defaults of ClusterConfig (types.hpp:83-94). */
void tsb_cluster_default(tsb_cluster* out);
/* ClusterConfig::validate (types.cpp:56-71). */
tsb_status tsb_cluster_validate(const tsb_cluster* c);
/* config_fingerprint (engine.hpp:68-74, engine.cpp:500-534): byte-wise FNV-1a-64 over the     */
/* config fields in declaration order, then the policy and the seed (enums one byte each).    */
uint64_t tsb_config_fingerprint(const tsb_cluster* c, int policy, uint64_t seed);

/* ------------------------------------------------------------------------------------ */
/* KV geometry and chunk plan (types.cpp:73-118)                                           */
/* ------------------------------------------------------------------------------------ */
typedef struct {
  int64_t layers;       /* L */
  int64_t kv_heads;     /* H (all ranks) */
  int64_t head_dim;     /* D */
  int64_t dtype_bytes;  /* E (2 = bf16) */
  int64_t chunk_tokens; /* KVBlock tokens = ClusterConfig::block_size_tokens (256) */
  int64_t page_tokens;  /* vLLM block_size (16) */
  int64_t tp_size;      /* KV-head shards; H % tp_size == 0 */
  int64_t tp_rank;      /* this GPU keeps heads [tp_rank*H/tp_size, (tp_rank+1)*H/tp_size) */
} tsb_kv_shape;

/* kv_bytes_per_token (types.cpp:113-118): 2*L*H*D*E; VALIDATION if any arg < 1. */
tsb_status tsb_kv_bytes_per_token(int64_t layers, int64_t kv_heads, int64_t head_dim,
                                  int64_t dtype_bytes, int64_t* out);
/* Validates a shape; returns full chunk bytes (L*2*C*H*D*E, the L2 slot size), local page
 * bytes (one page across all layers, K and V, this rank's heads) and local chunk bytes. */
tsb_status tsb_kv_shape_info(const tsb_kv_shape* s, int64_t* chunk_bytes,
                             int64_t* local_page_bytes, int64_t* local_chunk_bytes);

/* Struct-of-arrays queue of tiersim::RequestSpec (types.hpp:52-64). */
enum { TSB_HAS_DEADLINE = 1, TSB_HAS_MEASURED = 2 };
typedef struct {
  const int64_t* id;
  const double* arrival;
  const int64_t* context_tokens;
  const int64_t* query_tokens;
  const double* cache_hit_ratio;
  const uint8_t* flags; /* TSB_HAS_DEADLINE | TSB_HAS_MEASURED */
  const double* deadline;
  const double* measured_t_load;
  const double* measured_t_comp;
} tsb_queue;

/* RequestSpec::validate (types.cpp:40-54) for entry i. */
tsb_status tsb_request_validate(const tsb_queue* q, int64_t i);
/* cached_token_count / compute_token_count / derive_block_plan (types.cpp:73-101) for
 * entry i: the plan is n_blocks full chunks of block_tokens tokens and block_bytes bytes. */
tsb_status tsb_derive_block_plan(const tsb_queue* q, int64_t i, const tsb_cluster* c,
                                 int64_t* cached_tokens, int64_t* compute_tokens,
                                 int64_t* n_blocks, int64_t* block_tokens,
                                 int64_t* block_bytes);

/* ------------------------------------------------------------------------------------ */
/* Synthetic request stream (workload.cpp:31-36, 70-135; rng.hpp:19-70): the product's own  */
/* generate_workload / solo_baseline_ttft / assign_slos, bit-identical to the reference's.  */
/* ------------------------------------------------------------------------------------ */
typedef struct {
  int64_t num_requests;       /* DatasetProfile (workload.hpp:19-28) */
  double context_tokens_mean;
  double context_tokens_cv;
  double query_tokens_mean;
  double query_tokens_cv;
  double qps;                 /* WorkloadSpec (workload.hpp:55-68) */
  int64_t count;              /* 0 = num_requests */
  int32_t hit_kind;           /* HitRatioSource: 0 Fixed, 1 UniformChoice */
  double hit_fixed;
  const double* hit_choices;
  int64_t n_hit_choices;
  uint64_t seed;
} tsb_workload_spec;
/* builtin_profile("loogle" | "icl" | "code") into the profile fields (others defaulted:
 * qps 1, count 0, fixed hit 1.0, seed 0); TSB_UNKNOWN_PROFILE otherwise. */
tsb_status tsb_builtin_profile(const char* name, tsb_workload_spec* out);
tsb_status tsb_workload_validate(const tsb_workload_spec* w);
int64_t tsb_workload_count(const tsb_workload_spec* w);
/* generate_workload (workload.cpp:70-99): ids 1..n, Poisson arrivals, lognormal lengths. */
tsb_status tsb_generate_workload(const tsb_workload_spec* w, int64_t cap, int64_t* id,
                                 double* arrival, int64_t* context_tokens,
                                 int64_t* query_tokens, double* cache_hit_ratio, int64_t* n_out);
/* solo_baseline_ttft (workload.cpp:101-115) of entry i: its TTFT alone in an empty system. */
tsb_status tsb_solo_baseline_ttft(const tsb_queue* q, int64_t i, const tsb_cluster* c,
                                  double* ttft);
/* assign_slos (workload.cpp:117-135): deadline_out[i] = arrival + factor * solo baseline. */
tsb_status tsb_assign_slos(int64_t n, const tsb_queue* q, const tsb_cluster* c,
                           const double* factors, int64_t n_factors, uint64_t seed,
                           double* deadline_out);

/* ------------------------------------------------------------------------------------ */
/* Cost model (cost_model.cpp:14-85)                                                      */
/* models[4] = {load.slope, load.intercept, comp.slope, comp.intercept}                    */
/* ------------------------------------------------------------------------------------ */
void tsb_cost_models_from_config(const tsb_cluster* c, double models[4]);
double tsb_predict(double slope, double intercept, int64_t tokens);
tsb_status tsb_fit_linear(int64_t n, const int64_t* tokens, const double* seconds,
                          double* slope, double* intercept, int* slope_clamped,
                          int* intercept_clamped);
/* Scalar host forms for single-request callers (planning arithmetic, not the batched path):
 * estimate_service_cost (cost_model.cpp:56-71) and priority_key (scheduler.cpp:45-73) of
 * entry i.  tsb_priority_key returns MISSING_DEADLINE for EDF/LSTF without a deadline. */
tsb_status tsb_estimate_service_cost(const tsb_queue* q, int64_t i, const double models[4],
                                     const tsb_cluster* c, double* t_load, double* t_comp);
tsb_status tsb_priority_key(const tsb_queue* q, int64_t i, int policy, double t_load,
                            double t_comp, double* primary);

/* ------------------------------------------------------------------------------------ */
/* Batched scorer + schedule order (K4, K5).                                              */
/* Replaces estimate_service_cost (cost_model.cpp:56-71), priority_key (scheduler.cpp:45-73) */
/* and the pick_next drain (scheduler.cpp:75-100): order[k] is the queue index picked k-th. */
/* ------------------------------------------------------------------------------------ */
typedef enum {
  TSB_FIFO = 0,
  TSB_SJF_PT = 1,
  TSB_SJF_COST = 2,
  TSB_EDF = 3,
  TSB_LSTF = 4
} tsb_policy; /* PolicyKind order, scheduler.hpp:23 */

/* Device-pointer variant: every array in q and the outputs live in device memory.  Fully
 * asynchronous on `stream` except for the error check, which needs err_index: pass a host
 * pointer to get a synchronous check (MISSING_DEADLINE / VALIDATION with the first
 * offending queue index, as best_request_index would throw at scheduler.cpp:79-84), or
 * NULL to skip it (errors then surface at the next tsb_scorer_check). order may be NULL. */
typedef struct tsb_scorer tsb_scorer;
tsb_status tsb_scorer_create(int device, int64_t capacity, tsb_scorer** out);
void tsb_scorer_destroy(tsb_scorer* s);
tsb_status tsb_score_queue_device(tsb_scorer* s, void* stream, int64_t n, const tsb_queue* q,
                                  int policy, const double models[4], const tsb_cluster* c,
                                  double* t_load, double* t_comp, double* primary,
                                  int64_t* order, int64_t* err_index);
tsb_status tsb_scorer_check(tsb_scorer* s, void* stream, int64_t* err_index);
/* Host-pointer variant (the drop-in for a CPU caller): copies q in, runs K4+K5, copies
 * the results out, synchronises.  Any output may be NULL. */
tsb_status tsb_score_queue(tsb_scorer* s, void* stream, int64_t n, const tsb_queue* q,
                           int policy, const double models[4], const tsb_cluster* c,
                           double* t_load, double* t_comp, double* primary, int64_t* order);

/* ------------------------------------------------------------------------------------ */
/* Prefix chunk hasher (K3).  Definition in oracle/tsb_oracle.c (orc_hash_prefix_chunks);   */
/* the reference's only hash primitive is FNV-1a-64 (engine.cpp:500-534).                   */
/* Request r owns tokens [offsets[r], offsets[r+1]) and writes floor(len/256) chained chunk */
/* hashes at out[chunk_offsets[r] ...].  Device variants read only offsets[r] (the first     */
/* token) and chunk_offsets (the full-chunk counts), so requests may sit at padded, 16-byte  */
/* aligned starts with gaps between them: aligned leaves load as whole 16-byte vectors.      */
/* ------------------------------------------------------------------------------------ */
/* Measurement knob: phase-1 CTAs per SM (0 = default 3). */
tsb_status tsb_hash_set_grid(int ctas_per_sm);
/* Measurement knobs: phase-1 L2 prefetch distance in warp groups (0 = off, default 1); chain */
/* fused into phase 1 (1) or a separate pass (0, default).  -1 keeps the current setting.     */
tsb_status tsb_hash_set_tuning(int prefetch_groups, int fused_chain);
/* Phase 1 alone: each full chunk's own digest (no chain) at out[chunk_offsets[r] + c]. */
tsb_status tsb_hash_chunk_digests_device(void* stream, int64_t n_req, const int64_t* offsets,
                                         const int32_t* tokens, const int64_t* chunk_offsets, uint64_t* out);
tsb_status tsb_hash_prefix_chunks_device(void* stream, int64_t n_req, const int64_t* offsets,
                                         const int32_t* tokens, const int64_t* chunk_offsets,
                                         uint64_t* out);
/* Host-pointer variant: H2D tokens, hash, D2H hashes, synchronise. */
tsb_status tsb_hash_prefix_chunks(void* stream, int64_t n_req, const int64_t* offsets,
                                  const int32_t* tokens, uint64_t* out, int64_t* n_hashes);
/* Synthetic token ids on device (harness; same generator as orc_gen_tokens). */
tsb_status tsb_gen_tokens_device(void* stream, uint64_t seed, int64_t n_req,
                                 const int64_t* offsets, const int64_t* doc,
                                 const int64_t* shared_len, int32_t* out);

/* ------------------------------------------------------------------------------------ */
/* L2 chunk index (K7): chained prefix-chunk hash -> L2 pool slot, an open-addressing table   */
/* in HBM.  Replaces the synthetic cache_hit_ratio input of cached_token_count               */
/* (types.cpp:73-79) with a real prefix match: request r's matched prefix = the number of     */
/* leading chunks whose hash is indexed (hash c names the prefix [0, 256(c+1)), so the match  */
/* stops at the first absent chunk).  Hash values 2^64-1 and 2^64-2 are reserved.            */
/* ------------------------------------------------------------------------------------ */
typedef struct tsb_index tsb_index;
/* capacity is rounded up to a power of two; keep the load factor below ~0.5. */
tsb_status tsb_index_create(int device, int64_t capacity, tsb_index** out);
void tsb_index_destroy(tsb_index* x);
int64_t tsb_index_capacity(const tsb_index* x);
/* Device pointers; async.  Re-inserting an indexed hash updates its slot; when one batch holds
 * the same hash more than once, the lowest batch index wins (deterministic). */
tsb_status tsb_index_insert_device(tsb_index* x, void* stream, int64_t n, const uint64_t* hashes,
                                   const int64_t* slots);
tsb_status tsb_index_erase_device(tsb_index* x, void* stream, int64_t n, const uint64_t* hashes);
/* chunk_offsets[n_req+1] as for the hasher; slots_out[c] = the value inserted for chunk c (a pool
 * slot, or ~slot for a chunk held in the HBM tier: tsb_ingest_tiered / tsb_stage_set_hbm_tier
 * take it as is) for the matched prefix, -1 from the first miss on; matched_out[r] = matched
 * chunks of request r (authoritative: a stored value may itself be negative). */
tsb_status tsb_index_lookup_device(tsb_index* x, void* stream, int64_t n_req,
                                   const int64_t* chunk_offsets, const uint64_t* hashes,
                                   int64_t* slots_out, int64_t* matched_out);
/* Live entries and failed inserts (table full); synchronises. */
tsb_status tsb_index_stats(tsb_index* x, void* stream, int64_t* live, int64_t* full_failures);
/* Drop every entry (synchronous on `stream` order only). */
tsb_status tsb_index_clear(tsb_index* x, void* stream);
/* Rebuild the table without the tombstones erases left (probe paths shorten again); reports how
 * many were reclaimed.  Synchronises.  The host tsb_index_insert compacts by itself when a batch
 * finds the table full and tombstones exist. */
tsb_status tsb_index_compact(tsb_index* x, void* stream, int64_t* tombstones_reclaimed);
/* Host-pointer variants (synchronise); insert returns CAPACITY if the table is full.
 * chunk_offsets[0] must be 0. */
tsb_status tsb_index_insert(tsb_index* x, void* stream, int64_t n, const uint64_t* hashes,
                            const int64_t* slots);
tsb_status tsb_index_lookup(tsb_index* x, void* stream, int64_t n_req, const int64_t* chunk_offsets,
                            const uint64_t* hashes, int64_t* slots_out, int64_t* matched_out);

/* ------------------------------------------------------------------------------------ */
/* L2 chunk pool: pinned, portable, mapped host memory (replaces TierLedger(L2) as a byte   */
/* store; engine.cpp:18-49 stays the accounting).  Slot s holds one full chunk             */
/* [L][2][C][H][D] at host address base + s*chunk_bytes.                                   */
/* ------------------------------------------------------------------------------------ */
typedef struct tsb_pool tsb_pool;
tsb_status tsb_pool_create(const tsb_kv_shape* shape, int64_t n_slots, tsb_pool** out);
/* Adopt caller-owned memory instead (must be page-locked, e.g. cudaHostRegister'ed). */
tsb_status tsb_pool_wrap(const tsb_kv_shape* shape, void* host_base, int64_t n_slots,
                         tsb_pool** out);
/* Page-lock caller memory (cudaHostRegister portable|mapped), e.g. a shared-memory segment
 * every per-GPU process maps, so all GPUs of a box read one L2 pool; unregistered on destroy. */
tsb_status tsb_pool_register(const tsb_kv_shape* shape, void* host_base, int64_t n_slots,
                             tsb_pool** out);
/* NUMA-placed pool: anonymous memory bound to `numa_node` (mbind MPOL_BIND; -1 = default
 * policy), transparent huge pages advised, then page-locked portable|mapped.  One per GPU on the
 * GPU's own socket (tsb_device_numa_node) keeps each host link reading local DIMMs; the
 * reference's single L2 capacity (ClusterConfig::l2_capacity, types.hpp:88) becomes per-socket
 * shard pools of one rank's KV heads each.  munmap'ed on destroy. */
tsb_status tsb_pool_create_numa(const tsb_kv_shape* shape, int64_t n_slots, int numa_node,
                                tsb_pool** out);
/* NUMA node backing the pool's first page (get_mempolicy), -1 if unknown or a device pool. */
int tsb_pool_numa_node(const tsb_pool* p);
/* NUMA node of a GPU's PCIe root (sysfs numa_node of its bus id), -1 if unknown. */
int tsb_device_numa_node(int device);
void tsb_pool_destroy(tsb_pool* p);
void* tsb_pool_slot_ptr(tsb_pool* p, int64_t slot);
int64_t tsb_pool_slots(const tsb_pool* p);
int64_t tsb_pool_chunk_bytes(const tsb_pool* p);
/* Harness: fill slots [first, first+n) with the synthetic bf16 pattern (orc_synth_word)
 * from a device kernel writing through the mapped pointer; synchronises. */
tsb_status tsb_pool_fill_synthetic(tsb_pool* p, uint64_t seed, int64_t first, int64_t n,
                                   void* stream);

/* Peer-HBM tier: a chunk pool resident in GPU memory -- this GPU's or
 * a peer's over NVLink / NVSwitch -- with the same slot layout.  It stands where the reference
 * runs the L3->L2 network stage (engine.cpp:405-425): chunks another GPU already holds are
 * read peer-to-peer by the ingest kernels instead of crossing the host link.  Ingest from a
 * device pool runs K1 (SM loads; AUTO resolves to it) with the HBM grid, or K1b; CE is
 * UNSUPPORTED.  tsb_pool_slot_ptr returns the device address for these pools. */
typedef enum { TSB_POOL_HOST = 0, TSB_POOL_DEVICE = 1 } tsb_pool_location;
/* cudaMalloc n_slots chunks on `device` (owned; freed on destroy). */
tsb_status tsb_pool_create_device(int device, const tsb_kv_shape* shape, int64_t n_slots,
                                  tsb_pool** out);
/* Adopt caller-owned device memory of `device` (not freed on destroy). */
tsb_status tsb_pool_wrap_device(int device, const tsb_kv_shape* shape, void* dev_base,
                                int64_t n_slots, tsb_pool** out);
/* Export a tsb_pool_create_device pool to other processes: writes a 64-byte
 * cudaIpcMemHandle_t to handle_out. */
tsb_status tsb_pool_ipc_handle(const tsb_pool* p, void* handle_out);
/* Map a peer process's exported pool into this process (cudaIpcOpenMemHandle with lazy peer
 * access); `owner_device` is the pool's device ordinal as this process numbers it (for the
 * peer-access check; -1 = unknown).  Closed on destroy. */
tsb_status tsb_pool_open_ipc(const tsb_kv_shape* shape, const void* handle, int owner_device,
                             int64_t n_slots, tsb_pool** out);
/* Enable peer access from `device` to `peer` (idempotent); UNSUPPORTED when the pair cannot. */
tsb_status tsb_enable_peer_access(int device, int peer);
int tsb_pool_location_of(const tsb_pool* p);
int tsb_pool_device(const tsb_pool* p);

/* ------------------------------------------------------------------------------------ */
/* L1 paged allocator + block_table.                                                        */
/* Byte accounting is exactly TierLedger (engine.cpp:18-49): a chunk reservation is        */
/* granted iff no older reservation waits and it fits, else deferred; releases grant FIFO. */
/* Capacity = num_pages * local_page_bytes.  On grant the chunk's pages are taken from a   */
/* FIFO free list and written into block_table[row(request)][chunk*pages_per_chunk + j].   */
/* The KV arena is per layer [2][num_pages][page_tokens][H_local][D] (vLLM flash-attn).     */
/* ------------------------------------------------------------------------------------ */
typedef struct tsb_l1 tsb_l1;
typedef struct {
  int64_t request_id;
  int32_t block_index;
  int32_t bt_row; /* -1 for the standalone byte ledger */
  int64_t bytes;
} tsb_grant;

/* Standalone byte ledger: TierLedger (engine.hpp:22-53) with identical decisions and messages;
 * the L1 allocator below runs the same ledger object.  tier: 0 L3, 1 L2, 2 L1. */
typedef struct tsb_ledger tsb_ledger;
tsb_status tsb_ledger_create(int tier, int64_t capacity, tsb_ledger** out);
void tsb_ledger_destroy(tsb_ledger* l);
tsb_status tsb_ledger_request(tsb_ledger* l, int64_t request_id, int32_t block_index,
                              int64_t bytes, int* granted);
/* TierLedger::release: grants are written to out[0..min(n,cap)). */
tsb_status tsb_ledger_release(tsb_ledger* l, int64_t bytes, tsb_grant* out, int64_t cap,
                              int64_t* n);
int64_t tsb_ledger_reserved(const tsb_ledger* l);
int64_t tsb_ledger_capacity(const tsb_ledger* l);
int64_t tsb_ledger_deferred(const tsb_ledger* l);

/* arena: device pointer of L*2*num_pages*page_tokens*H_local*D*E bytes, or NULL to allocate
 * internally.  max_rows = concurrent requests; max_chunks = chunk columns per row. */
tsb_status tsb_l1_create(int device, const tsb_kv_shape* shape, int64_t num_pages,
                         int64_t max_rows, int64_t max_chunks, void* arena, tsb_l1** out);
void tsb_l1_destroy(tsb_l1* l1);
/* Physical layout of each layer's pages, the consumer's KV-cache layout (installed vLLM 0.22:
 * v1/attention/backends/flash_attn.py:140-149 and flashinfer.py:357-389).  Same bytes per page;
 * only the addresses differ.  Default FLASH_ATTN. */
typedef enum {
  TSB_LAYOUT_FLASH_ATTN = 0,    /* layer = [2][pages][P][H_local][D]  (K and V planes)      */
  TSB_LAYOUT_FLASHINFER_NHD = 1, /* layer = [pages][2][P][H_local][D]  (page-major, NHD)     */
  TSB_LAYOUT_FLASHINFER_HND = 2  /* layer = [pages][2][H_local][P][D]  (page-major, HND)     */
} tsb_kv_layout;
/* Sets the page layout; VALIDATION unless nothing is reserved yet. */
tsb_status tsb_l1_set_layout(tsb_l1* l1, int layout);
int tsb_l1_layout(const tsb_l1* l1);
/* TierLedger::request (engine.cpp:22-36).  bytes must be a whole number of local pages
 * (a chunk: chunk_tokens * local bytes/token).  *granted = 1 when granted now; *bt_row gets
 * the request's block_table row (assigned at its first reservation). */
tsb_status tsb_l1_request(tsb_l1* l1, int64_t request_id, int32_t block_index, int64_t bytes,
                          int* granted, int32_t* bt_row);
/* Releases every page of a request (ComputeDone release, engine.cpp:280-282) and grants
 * waiting reservations FIFO while they fit (TierLedger::release, engine.cpp:38-49).  The
 * grants are written to out[0..min(n,cap)). */
tsb_status tsb_l1_release_request(tsb_l1* l1, int64_t request_id, tsb_grant* out, int64_t cap,
                                  int64_t* n);
int64_t tsb_l1_reserved(const tsb_l1* l1);
int64_t tsb_l1_capacity(const tsb_l1* l1);
int64_t tsb_l1_deferred(const tsb_l1* l1);
int64_t tsb_l1_free_pages(const tsb_l1* l1);
int64_t tsb_l1_num_pages(const tsb_l1* l1);
int64_t tsb_l1_page_bytes(const tsb_l1* l1);
int tsb_l1_device(const tsb_l1* l1);
tsb_status tsb_l1_shape(const tsb_l1* l1, tsb_kv_shape* out);
void* tsb_l1_arena(tsb_l1* l1);
void* tsb_l1_layer_ptr(tsb_l1* l1, int64_t layer);
/* Host (pinned) mirror of the block table, [max_rows][max_chunks*pages_per_chunk] int32,
 * -1 = unassigned, and its device copy. */
const int32_t* tsb_l1_block_table_host(const tsb_l1* l1);
const int32_t* tsb_l1_block_table_device(const tsb_l1* l1);
int64_t tsb_l1_block_table_stride(const tsb_l1* l1);
/* Copies the host block table to the device copy on `stream` (async). */
tsb_status tsb_l1_sync_block_table(tsb_l1* l1, void* stream);

/* ------------------------------------------------------------------------------------ */
/* L2 -> L1 ingest (K1 / K1b / CE+K2).  The real pcie_dispatch hop (engine.cpp:427-446,     */
/* duration model engine.cpp:206-207).  One call moves every (item, layer in               */
/* [layer_lo, layer_hi)) of the batch, layer by layer.  layer_events (NULL, or an array of  */
/* layer_hi-layer_lo cudaEvent_t passed as void*, entries may be NULL): event k is recorded */
/* on `stream` once layer layer_lo+k of every item is resident in L1 -- the per-layer fence */
/* a prefill consumer waits on with cudaStreamWaitEvent.                                    */
/* ------------------------------------------------------------------------------------ */
typedef struct {
  int64_t src_slot;    /* L2 pool slot holding the chunk */
  int32_t bt_row;      /* block_table row of the owning request */
  int32_t chunk_index; /* KVBlock::block_index within the request */
} tsb_ingest_item;

typedef enum {
  TSB_INGEST_AUTO = 0,     /* host pool: CE for full-head shapes and for head-sharded item
                              lists whose consecutive-slot runs carry >= 3.1 MB per copy,
                              else ZEROCOPY; device pool or device items: ZEROCOPY */
  TSB_INGEST_ZEROCOPY = 1, /* K1: SM 16B loads from mapped host memory, scatter to pages */
  TSB_INGEST_BULK = 2,     /* K1b: one tensor-map TMA load (UTMALDG) per page segment into a
                              shared-memory ring, one cp.async.bulk store per segment; NHD via a
                              2D map, HND via a 3D (D, rows, heads) map that transposes */
  TSB_INGEST_CE = 3,       /* copy engine H2D into an HBM staging ring, then K2 scatter;
                              host reads run on an internal copy stream ordered after the
                              work queued on `stream` before the call.  Consecutive layers up
                              to the next requested fence share a staging group when they
                              fit.  Head-sharded shapes copy only this rank's heads: one
                              strided cudaMemcpy3DAsync per run of consecutive slots per
                              group.  K2 runs on an internal greatest-priority stream */
  TSB_INGEST_CE_DIRECT = 4 /* copy engines straight into the pages, no SM work at all: one
                              cudaMemcpy3DAsync per (item, run of consecutive pages) covering
                              K|V x the layers up to the next requested fence; for full-head
                              chunks into flash-attn / NHD pages (the page segment is
                              contiguous on both sides), else UNSUPPORTED */
} tsb_ingest_mode;

/* One pcie_dispatch with real bytes (engine.cpp:427-446; PcieDone engine.cpp:258-272).
 * items: host array (copied into a pinned ring internally, so it may be reused on return).
 * All grants for the items must already be in the block table (tsb_l1_sync_block_table).
 * VALIDATION if an item's slot, row or chunk index is outside the pool / block table. */
tsb_status tsb_ingest(tsb_l1* l1, tsb_pool* pool, const tsb_ingest_item* items, int64_t n_items,
                      int64_t layer_lo, int64_t layer_hi, int mode, void* stream,
                      void* const* layer_events);
/* Two-tier ingest: an item with src_slot < 0 names slot ~src_slot of hbm_pool (a chunk already
 * resident in this GPU's or a peer's HBM -- the peer-HBM tier that stands in for the L3->L2
 * network stage, engine.cpp:405-425); the others name slots of pool.  The HBM-tier items are
 * moved by K1 (HBM / NVLink speed) on an internal stream beside the host part (`mode`), so the
 * link never waits for them; layer_events and later work on `stream` cover both. */
tsb_status tsb_ingest_tiered(tsb_l1* l1, tsb_pool* pool, tsb_pool* hbm_pool,
                             const tsb_ingest_item* items, int64_t n_items, int64_t layer_lo,
                             int64_t layer_hi, int mode, void* stream, void* const* layer_events);
/* The kernel path tsb_ingest takes for these items and mode (AUTO resolved; other modes returned
 * as given) -- which mechanism carries the pcie_dispatch hop (engine.cpp:427-446).  items: host
 * array or NULL (device items). */
/* 1 if TSB_INGEST_CE_DIRECT can serve this L1 / pool pair (full heads, host pool, flash-attn or
 * NHD pages).  The load stage uses it whenever a prefill shares the GPU, so ingest needs no SMs. */
int tsb_ingest_ce_direct_supported(const tsb_l1* l1, const tsb_pool* pool);
tsb_status tsb_ingest_resolve_mode(const tsb_l1* l1, const tsb_pool* pool,
                                   const tsb_ingest_item* items, int64_t n_items, int mode,
                                   int* resolved);
/* Device-items variant (items already in device memory; CE mode needs host items and returns
 * UNSUPPORTED here).  The items are not range-checked: the caller guarantees them. */
tsb_status tsb_ingest_device(tsb_l1* l1, tsb_pool* pool, const tsb_ingest_item* items_dev,
                             int64_t n_items, int64_t layer_lo, int64_t layer_hi, int mode,
                             void* stream, void* const* layer_events);
/* K2 alone: scatter chunks already staged in HBM: item i's layers [layer_lo, layer_hi), laid out
 * as in the chunk ([layer][K/V][token][kv_head][dim]), start at staging + i*(hi-lo)*2*C*H*D*E
 * (src_slot is ignored). */
tsb_status tsb_scatter_device(tsb_l1* l1, const void* staging, const tsb_ingest_item* items_dev,
                              int64_t n_items, int64_t layer_lo, int64_t layer_hi, void* stream);
/* K2 alone on the CE path's staging format: item i's layers [layer_lo, layer_hi) of this rank's
 * heads only, packed [layer][K/V][C][H_local][D], at staging + i*(hi-lo)*2*C*H_local*D*E. */
tsb_status tsb_scatter_device_packed(tsb_l1* l1, const void* staging,
                                     const tsb_ingest_item* items_dev, int64_t n_items,
                                     int64_t layer_lo, int64_t layer_hi, void* stream);
/* Chunk replication inside L1 (K8): a chunk resident in one request's pages copied into another
 * request's granted pages, HBM -> HBM, for layers [layer_lo, layer_hi) -- instead of moving the
 * same L2 chunk over the host link again (LooGLE-like batches read each document chunk from many
 * requests).  Both rows' pages must be granted and the source's bytes written by work already
 * queued on `stream`.  Items are range-checked; async. */
typedef struct {
  int32_t src_row, src_chunk; /* block_table row / chunk index holding the bytes */
  int32_t dst_row, dst_chunk; /* where they go */
} tsb_page_copy;
tsb_status tsb_l1_copy_chunks(tsb_l1* l1, const tsb_page_copy* items, int64_t n_items, int64_t layer_lo,
                              int64_t layer_hi, void* stream);
/* Tuning knobs for measurement (0 = default); no reference counterpart (the reference models
 * the hop's cost only, engine.cpp:206-207). */
tsb_status tsb_ingest_set_grid(int zerocopy_ctas, int bulk_ctas, int scatter_ctas);
/* K2 implementation: 0 = SM 16-byte load/store warps (default), 1 = cp.async.bulk ring. */
tsb_status tsb_ingest_set_scatter(int impl, int ctas);
/* CE copy strategy: 0 = one cudaMemcpyAsync per (item, layer span), 1 = one cudaMemcpy2DAsync
 * per run of consecutive pool slots (default).  Full-head shapes only; head-sharded shapes
 * always use one 3D copy per consecutive-slot run.  (The batched-memcpy entry points are not
 * used: they are closed on this GPU pool after GPU faults.)
 * staging_bytes: HBM staging ring size (0 = default 1 GiB, two halves). */
tsb_status tsb_ingest_set_ce(int variant, int64_t staging_bytes);
/* Per-L1 cap on one CE staging group (bytes of one half of the ring a group may fill; 0 = the
 * whole half).  Smaller groups shorten each copy-engine wait that a scatter launch sits behind;
 * the load stage sets it while a prefill shares the GPU (tsb_stage_options.prefill or a hook). */
tsb_status tsb_l1_set_ce_group_bytes(tsb_l1* l1, int64_t bytes);
int64_t tsb_l1_ce_group_bytes(const tsb_l1* l1);

/* ------------------------------------------------------------------------------------ */
/* Load stage: the real-time L2->L1 dispatcher.  Follows SimEngine's dispatch semantics    */
/* (engine.cpp:290-302 pump, :341-355 admit, :405-425 proactive L1 reservation at dispatch, */
/* :427-446 pcie_dispatch, :258-272 PcieDone, :280-282 L1 release at ComputeDone) with real */
/* bytes and real time: requests are scored and ordered on the GPU (K4/K5), admitted in     */
/* pick order, every planned chunk reserves L1 pages through the TierLedger-semantics        */
/* allocator (grant-before-hop; deferred reservations are granted FIFO as earlier requests  */
/* release), granted chunks are ingested per request in pick order, and a request's pages   */
/* are released when its ingest (and optional synthetic prefill) completes.                 */
/* ------------------------------------------------------------------------------------ */
typedef struct tsb_stage tsb_stage;

typedef struct {
  int32_t mode;         /* tsb_ingest_mode */
  int32_t policy;       /* tsb_policy used for the admission (pick) order */
  int32_t layer_events; /* 1: per-layer fences per request (layer-pipelined prefill) */
  int32_t prefill;      /* 1: synthetic prefill K6 per request after/with its ingest, lasting
                           compute_base + compute_per_token*n + compute_quadratic*n^2 seconds
                           (engine.cpp:210-212); 0: pages are released once resident */
  int32_t prefill_ctas; /* CTAs per K6 launch (0 = 148) */
  int32_t record_trace; /* 1: keep TraceEvent-schema rows (events.hpp:33-42) for the run */
  uint64_t verify_seed; /* harness check, 0 = off: before a request's pages are released, count
                           page words differing from tsb_pool_fill_synthetic(verify_seed) */
  int32_t pace_network; /* online mode with an L3 store: a network hop lasts at least
                           transfer_base_latency + bytes / network_bandwidth (engine.cpp:205) */
  int32_t reuse_l1;     /* a chunk whose L2 slot is already resident in another live request's
                           pages (its hop issued) is replicated HBM -> HBM (K8) instead of
                           crossing the link again; the holder's release waits for the copies.
                           Batch and online modes; TSB_UNSUPPORTED with an L3 store */
} tsb_stage_options;

typedef struct {
  int64_t request_id;
  int32_t pick_position;   /* index in the admission order */
  int32_t deferred_chunks; /* chunk reservations that waited for a release */
  int64_t chunks;          /* chunks ingested (derive_block_plan size) */
  int64_t bytes;           /* bytes moved L2 -> L1 for this request on this GPU */
  double first_layer_ms;   /* run start -> layer lo of every chunk resident (CUDA events) */
  double resident_ms;      /* run start -> all layers resident (Timestamps::l1_resident) */
  double done_ms;          /* run start -> prefill done / pages released (first token) */
  double admit_ms;         /* run start -> admitted (Timestamps::scheduled; host clock) */
  double arrival_ms;       /* run start -> arrival (online mode: replayed arrival time) */
  double ingest_begin_ms;  /* run start -> its first L2 -> L1 hop began (CUDA event); with
                              resident_ms the measured T_load sample for fit_linear */
  int64_t cached_tokens;   /* cached_token_count (types.cpp:73-79): the T_load regressor */
  int64_t compute_tokens;  /* compute_token_count (types.cpp:81-83): the T_comp regressor */
} tsb_stage_request;

typedef struct {
  int64_t bytes;           /* total bytes delivered into L1 pages (host link + HBM tier + reuse_l1
                              replication; the link part is bytes - reused_chunks * chunk bytes) */
  double device_ms;        /* first ingest start -> last request resident (CUDA events) */
  double wall_ms;          /* host wall time of tsb_stage_run */
  int64_t ingest_calls;
  int64_t deferred_chunks;
  int64_t releases;
  int64_t kernel_launches; /* libtsb kernels launched during the run */
  uint64_t verify_mismatches; /* with verify_seed != 0 */
  int64_t net_blocks;      /* online mode with an L3 store: L3 -> L2 network hops */
  int64_t l2_deferred;     /* ... L2 reservations that waited for a release (engine.cpp:357-362) */
  int64_t reused_chunks;   /* reuse_l1: chunks replicated from L1 instead of the host link */
} tsb_stage_stats;

/* TraceEvent row (events.hpp:33-42): kind 1 TransferDone, 2 AllocationGrant, 4 DispatchWake;
 * stage 1 Pcie, 2 Compute; tier 2 L1 (or -1); time in seconds from run start (host clock for
 * dispatch/grant rows, CUDA events for TransferDone rows). */
typedef struct {
  double time;
  uint64_t seq;
  int32_t kind;
  int32_t stage;
  int32_t tier;
  int32_t block_index;
  int64_t request_id;
  int64_t bytes;
} tsb_trace_row;

tsb_status tsb_stage_create(tsb_l1* l1, tsb_pool* pool, tsb_stage** out);
/* Online mode only: blocks start in the L3 store `l3` (a host pool of the same chunk geometry;
 * slots passed to tsb_stage_run_online name L3 chunks) and make the network hop L3 -> L2 for
 * real: the stage's pool becomes the L2 tier, a TierLedger(L2) over min(l2_capacity, slots)
 * whole slots with a FIFO slot free list (request_l2 at admit, engine.cpp:341-362; released when
 * the block's L2 -> L1 hop completes, :264); one block in flight, copied by `copy_threads` host
 * threads (engine.cpp:405-425).  NULL detaches.  tsb_stage_run returns UNSUPPORTED while set. */
tsb_status tsb_stage_set_l3(tsb_stage* s, tsb_pool* l3, int copy_threads);
/* Prefill consumer: called on the host for every layer of a request's prefill, after the stage
 * made the compute stream wait for that layer's fence; enqueue the layer's work on `stream` (the
 * stage's compute stream) and return 0.  Replaces the K6 timer (the reference's compute stage,
 * engine.cpp:448-473; ComputeDone = the stream passing the last layer).  NULL restores K6. */
typedef int (*tsb_prefill_hook)(void* user, int64_t q_index, int32_t bt_row, int64_t layer, void* stream);
tsb_status tsb_stage_set_prefill_hook(tsb_stage* s, tsb_prefill_hook hook, void* user);
/* The stage's compute stream (lowest priority; prefill runs here). */
void* tsb_stage_compute_stream(tsb_stage* s);
/* Run prefill on the caller's stream instead (not destroyed by the stage; NULL = a stage-owned
 * lowest-priority stream again): a consumer whose framework owns stream lifetimes (e.g. a torch
 * stream) keeps its work and host buffers tied to a stream that outlives the stage. */
tsb_status tsb_stage_set_compute_stream(tsb_stage* s, void* stream);
void tsb_stage_destroy(tsb_stage* s);
/* HBM tier of the stage (NULL clears it): in tsb_stage_run / _online, a slot < 0 names slot ~slot
 * of hbm_pool (same chunk geometry as the L2 pool); those chunks bypass the host link. */
tsb_status tsb_stage_set_hbm_tier(tsb_stage* s, tsb_pool* hbm_pool);
/* Runs one batch to completion (synchronises).  Request i's planned chunk c is stored in pool
 * slot slots[slot_offsets[i] + c]; slot_offsets has n+1 entries and each request must list
 * exactly derive_block_plan(spec_i).size() slots.  results may be NULL. */
tsb_status tsb_stage_run(tsb_stage* s, int64_t n, const tsb_queue* q, const tsb_cluster* c,
                         const double models[4], const int64_t* slot_offsets,
                         const int64_t* slots, const tsb_stage_options* opt, void* stream,
                         tsb_stage_request* results, tsb_stage_stats* stats);
/* Online replay: requests arrive at their arrival_time (seconds after the first arrival, on the
 * host clock) and the stage runs SimEngine's decoupled control loop in real time
 * (engine.cpp:290-302): the best pending request (PriorityKey order, keys from the GPU scorer)
 * is admitted only when the ingest stage is idle and has no backlog (try_admit, :318-339);
 * admission reserves L1 for its whole plan (proactive, :419); granted chunks are ingested in
 * admission order (pcie_dispatch, :427-446); the compute stage prefills the best-key resident
 * request whenever it is idle (try_start_compute, :448-473) with the K6 synthetic prefill
 * (compute_base + compute_per_token*n + compute_quadratic*n^2); pages are released at
 * ComputeDone (:280-282).  done_ms - arrival_ms is the request's TTFT.  opt->prefill is
 * ignored (always on).  Synchronises; results may be NULL. */
tsb_status tsb_stage_run_online(tsb_stage* s, int64_t n, const tsb_queue* q,
                                const tsb_cluster* c, const double models[4],
                                const int64_t* slot_offsets, const int64_t* slots,
                                const tsb_stage_options* opt, void* stream,
                                tsb_stage_request* results, tsb_stage_stats* stats);
/* Trace of the last run (when record_trace was set): copies min(n, cap) rows. */
tsb_status tsb_stage_trace(tsb_stage* s, tsb_trace_row* out, int64_t cap, int64_t* n);

/* Harness check: counts bytes of the items' pages (layers [lo,hi)) that differ from the
 * synthetic pattern of their source slot (as filled by tsb_pool_fill_synthetic with `seed`);
 * synchronises. */
tsb_status tsb_l1_verify_synthetic(tsb_l1* l1, const tsb_ingest_item* items, int64_t n_items,
                                   int64_t layer_lo, int64_t layer_hi, uint64_t seed,
                                   int64_t pool_chunk_bytes, void* stream, uint64_t* mismatches);

#ifdef __cplusplus
}
#endif
#endif
