/*
 * tsb_oracle.c — CPU restatement of the CALVO KV-ingest hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see tsb_oracle.h).  Each function cites the reference
 * file:line it restates; paths are relative to /root/reference/proj/.  Built with
 * -ffp-contract=off so every f64 expression is evaluated as written, in the
 * reference's operation order.
 */
#include "tsb_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define FNV_OFFSET 0xcbf29ce484222325ull /* engine.cpp:518 (config_fingerprint seed) */
#define FNV_PRIME 0x100000001b3ull       /* engine.cpp:504 (fnv1a multiplier) */

/* ------------------------------------------------------------------------ */
/* planning arithmetic                                                       */
/* ------------------------------------------------------------------------ */

/* core/src/types.cpp:113-118 */
int orc_kv_bytes_per_token(int64_t layers, int64_t kv_heads, int64_t head_dim,
                           int64_t dtype_bytes, int64_t* out) {
  if (layers < 1 || kv_heads < 1 || head_dim < 1 || dtype_bytes < 1) return ORC_VALIDATION;
  *out = 2 * layers * kv_heads * head_dim * dtype_bytes;
  return ORC_OK;
}

/* core/src/types.cpp:73-79: floor((double)ctx * hit / (double)block) * block */
int64_t orc_cached_token_count(int64_t context_tokens, double hit, int64_t block_size) {
  const double hit_tokens = (double)context_tokens * hit;
  const int64_t blocks = (int64_t)floor(hit_tokens / (double)block_size);
  return blocks * block_size;
}

/* core/src/types.cpp:81-83 */
int64_t orc_compute_token_count(int64_t context_tokens, int64_t query_tokens, double hit,
                                int64_t block_size) {
  return context_tokens + query_tokens - orc_cached_token_count(context_tokens, hit, block_size);
}

/* ------------------------------------------------------------------------ */
/* cost model                                                                */
/* ------------------------------------------------------------------------ */

/* core/src/cost_model.cpp:52-54 */
double orc_predict(double slope, double intercept, int64_t tokens) {
  return intercept + slope * (double)tokens;
}

/* core/src/cost_model.cpp:73-85; out = {load.slope, load.intercept, comp.slope, comp.intercept} */
void orc_cost_models_from_config(const orc_cluster* c, double out[4]) {
  const double bpt = (double)c->bytes_per_token;
  out[0] = bpt * (1.0 / c->network_bandwidth + 1.0 / c->pcie_bandwidth) +
           2.0 * c->transfer_base_latency / (double)c->block_size_tokens;
  out[1] = 0.0;
  out[2] = c->compute_per_token;
  out[3] = c->compute_base;
}

/* core/src/cost_model.cpp:14-50 */
int orc_fit_linear(int64_t n, const int64_t* tokens, const double* seconds, double* slope,
                   double* intercept, int* slope_clamped, int* intercept_clamped) {
  if (n < 2) return ORC_DEGENERATE_FIT;
  double mx = 0.0, my = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    mx += (double)tokens[i];
    my += seconds[i];
  }
  const double dn = (double)n;
  mx /= dn;
  my /= dn;
  double sxx = 0.0, sxy = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double dx = (double)tokens[i] - mx;
    sxx += dx * dx;
    sxy += dx * (seconds[i] - my);
  }
  if (sxx == 0.0) return ORC_DEGENERATE_FIT;
  double s = sxy / sxx;
  double b = my - s * mx;
  *slope_clamped = *intercept_clamped = 0;
  if (s < 0.0) { s = 0.0; *slope_clamped = 1; }
  if (b < 0.0) { b = 0.0; *intercept_clamped = 1; }
  *slope = s;
  *intercept = b;
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* scorer: estimate_service_cost (cost_model.cpp:56-71) + priority_key        */
/* (scheduler.cpp:39-73), evaluated in queue order so the first MissingDeadline */
/* is reported at the index best_request_index would throw at (:79-84).       */
/* ------------------------------------------------------------------------ */
int orc_score_queue(int64_t n, const orc_queue* q, int policy, const double m[4],
                    const orc_cluster* c, double* t_load, double* t_comp, double* primary,
                    int64_t* err_index) {
  *err_index = -1;
  for (int64_t i = 0; i < n; ++i) {
    double tl = 0.0, tc = 0.0;
    const uint8_t fl = q->flags[i];
    if (fl & ORC_HAS_MEASURED) {
      tl = q->measured_t_load[i];
      tc = q->measured_t_comp[i];
    } else {
      const int64_t cached =
          orc_cached_token_count(q->context_tokens[i], q->cache_hit_ratio[i], c->block_size_tokens);
      if (cached > 0) tl = orc_predict(m[0], m[1], cached);
      const int64_t ct = q->context_tokens[i] + q->query_tokens[i] - cached;
      tc = orc_predict(m[2], m[3], ct);
      if (c->compute_quadratic > 0.0) {
        const double dct = (double)ct;
        tc += c->compute_quadratic * dct * dct;
      }
    }
    double key = 0.0;
    switch (policy) {
      case ORC_FIFO: key = q->arrival[i]; break;
      case ORC_SJF_PT: {
        /* scheduler.cpp:39-43 */
        const double hit_tokens = floor((double)q->context_tokens[i] * q->cache_hit_ratio[i]);
        key = (double)(q->context_tokens[i] + q->query_tokens[i]) - hit_tokens;
        break;
      }
      case ORC_SJF_COST: key = tl + tc; break;
      case ORC_EDF:
        if (!(fl & ORC_HAS_DEADLINE)) { *err_index = i; return ORC_MISSING_DEADLINE; }
        key = q->deadline[i];
        break;
      case ORC_LSTF:
        if (!(fl & ORC_HAS_DEADLINE)) { *err_index = i; return ORC_MISSING_DEADLINE; }
        key = q->deadline[i] - (tl + tc);
        break;
      default: return ORC_VALIDATION;
    }
    t_load[i] = tl;
    t_comp[i] = tc;
    primary[i] = key;
  }
  return ORC_OK;
}

/* PriorityKey::operator< (scheduler.hpp:38-42) */
int orc_key_less(double pa, double aa, int64_t ia, double pb, double ab, int64_t ib) {
  if (pa != pb) return pa < pb;
  if (aa != ab) return aa < ab;
  return ia < ib;
}

/* Merge sort by PriorityKey::operator<.  With unique ids (engine.cpp:126-127) the
 * key is a total order, so this equals the pick_next drain (scheduler.cpp:93-100). */
int orc_sort_order(int64_t n, const double* p, const double* a, const int64_t* id,
                   int64_t* order) {
  int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  if (!tmp) return ORC_VALIDATION;
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  for (int64_t width = 1; width < n; width *= 2) {
    for (int64_t lo = 0; lo < n; lo += 2 * width) {
      int64_t mid = lo + width < n ? lo + width : n;
      int64_t hi = lo + 2 * width < n ? lo + 2 * width : n;
      int64_t i = lo, j = mid, k = lo;
      while (i < mid && j < hi) {
        const int64_t x = order[i], y = order[j];
        if (orc_key_less(p[y], a[y], id[y], p[x], a[x], id[x])) { tmp[k++] = y; ++j; }
        else { tmp[k++] = x; ++i; }
      }
      while (i < mid) tmp[k++] = order[i++];
      while (j < hi) tmp[k++] = order[j++];
    }
    memcpy(order, tmp, sizeof(int64_t) * (size_t)n);
  }
  free(tmp);
  return ORC_OK;
}

/* Repeated best_request_index + erase (scheduler.cpp:75-100): O(n^2), small n only. */
int orc_drain_order(int64_t n, const double* p, const double* a, const int64_t* id,
                    int64_t* order) {
  int64_t* q = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  if (!q) return ORC_VALIDATION;
  for (int64_t i = 0; i < n; ++i) q[i] = i;
  int64_t len = n;
  for (int64_t out = 0; out < n; ++out) {
    int64_t best = 0;
    for (int64_t i = 1; i < len; ++i) {
      const int64_t x = q[i], b = q[best];
      if (orc_key_less(p[x], a[x], id[x], p[b], a[b], id[b])) best = i;
    }
    order[out] = q[best];
    memmove(q + best, q + best + 1, sizeof(int64_t) * (size_t)(len - best - 1));
    --len;
  }
  free(q);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* TierLedger: engine.cpp:18-49 (byte ledger, strict-FIFO deferral)          */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t request_id;
  int32_t block_index;
  int64_t bytes;
} orc_pending;

struct orc_ledger {
  int64_t capacity, reserved;
  orc_pending* q;
  int64_t head, len, cap;
};

orc_ledger* orc_ledger_new(int64_t capacity) {
  if (capacity <= 0) return NULL; /* engine.cpp:18-20 ValidationError */
  orc_ledger* l = (orc_ledger*)calloc(1, sizeof(orc_ledger));
  l->capacity = capacity;
  l->cap = 16;
  l->q = (orc_pending*)malloc(sizeof(orc_pending) * (size_t)l->cap);
  return l;
}

void orc_ledger_free(orc_ledger* l) {
  if (!l) return;
  free(l->q);
  free(l);
}

static void ledger_push(orc_ledger* l, orc_pending p) {
  if (l->len == l->cap) {
    orc_pending* nq = (orc_pending*)malloc(sizeof(orc_pending) * (size_t)(l->cap * 2));
    for (int64_t i = 0; i < l->len; ++i) nq[i] = l->q[(l->head + i) % l->cap];
    free(l->q);
    l->q = nq;
    l->head = 0;
    l->cap *= 2;
  }
  l->q[(l->head + l->len) % l->cap] = p;
  ++l->len;
}

/* engine.cpp:22-36 */
int orc_ledger_request(orc_ledger* l, int64_t request_id, int32_t block_index, int64_t bytes,
                       int* granted) {
  if (bytes <= 0) return ORC_VALIDATION;
  if (bytes > l->capacity) return ORC_CAPACITY;
  if (l->len == 0 && l->reserved + bytes <= l->capacity) {
    l->reserved += bytes;
    *granted = 1;
    return ORC_OK;
  }
  orc_pending p = {request_id, block_index, bytes};
  ledger_push(l, p);
  *granted = 0;
  return ORC_OK;
}

/* engine.cpp:38-49 */
int orc_ledger_release(orc_ledger* l, int64_t bytes, int64_t* req_out, int32_t* blk_out,
                       int64_t* bytes_out, int64_t cap, int64_t* n_out) {
  *n_out = 0;
  if (bytes < 0 || bytes > l->reserved) return ORC_VALIDATION;
  l->reserved -= bytes;
  while (l->len > 0 && l->reserved + l->q[l->head].bytes <= l->capacity) {
    const orc_pending p = l->q[l->head];
    l->reserved += p.bytes;
    if (*n_out < cap) {
      req_out[*n_out] = p.request_id;
      blk_out[*n_out] = p.block_index;
      bytes_out[*n_out] = p.bytes;
    }
    ++*n_out;
    l->head = (l->head + 1) % l->cap;
    --l->len;
  }
  return ORC_OK;
}

int64_t orc_ledger_reserved(const orc_ledger* l) { return l->reserved; }
int64_t orc_ledger_deferred(const orc_ledger* l) { return l->len; }

/* ------------------------------------------------------------------------ */
/* alloc_ref: deterministic FIFO free list of page ids.  No reference          */
/* counterpart (the reference ledger only counts bytes, engine.cpp:18-49); the */
/* ledger decides WHEN a chunk is granted, this decides WHICH pages it gets:   */
/* pages are taken from the front in ascending order initially and returned to */
/* the back in release order.                                                 */
/* ------------------------------------------------------------------------ */
struct orc_pages {
  int32_t* ring;
  int64_t cap, head, len;
};

orc_pages* orc_pages_new(int64_t num_pages) {
  orc_pages* p = (orc_pages*)calloc(1, sizeof(orc_pages));
  p->cap = num_pages;
  p->ring = (int32_t*)malloc(sizeof(int32_t) * (size_t)(num_pages > 0 ? num_pages : 1));
  for (int64_t i = 0; i < num_pages; ++i) p->ring[i] = (int32_t)i;
  p->len = num_pages;
  return p;
}

void orc_pages_free(orc_pages* p) {
  if (!p) return;
  free(p->ring);
  free(p);
}

int64_t orc_pages_take(orc_pages* p, int64_t n, int32_t* out) {
  if (n > p->len) return -1;
  for (int64_t i = 0; i < n; ++i) out[i] = p->ring[(p->head + i) % p->cap];
  p->head = (p->head + n) % p->cap;
  p->len -= n;
  return n;
}

void orc_pages_give(orc_pages* p, int64_t n, const int32_t* ids) {
  for (int64_t i = 0; i < n; ++i) p->ring[(p->head + p->len + i) % p->cap] = ids[i];
  p->len += n;
}

int64_t orc_pages_available(const orc_pages* p) { return p->len; }

/* ------------------------------------------------------------------------ */
/* scatter_ref: the L2->L1 hop as bytes.  The reference models it only as a   */
/* duration (engine.cpp:206-207, dispatched by pcie_dispatch :427-446); here   */
/* each full chunk of the plan (types.cpp:85-101) is copied page by page from  */
/* the chunk layout [L][2][C][H][D] into the paged layout [L][2][pages][P][Hl][D] */
/* through block_table.  TP rank r keeps heads [r*Hl, (r+1)*Hl).               */
/* ------------------------------------------------------------------------ */
/* layout (the consumer's KV-cache layout, installed vLLM 0.22):                 */
/*   0 flash-attn   layer = [2][pages][P][Hl][D]  (v1/attention/backends/flash_attn.py:140-149) */
/*   1 FlashInfer   layer = [pages][2][P][Hl][D]  (flashinfer.py:357-368, NHD order :380-381)  */
/*   2 FlashInfer   layer = [pages][2][Hl][P][D]  (HND stride order, flashinfer.py:385-386)    */
/* arena_layer0: the arena buffer starts at layer arena_layer0 (a window of layers; 0 = whole). */
static void scatter_ref_impl(const orc_kv_shape* s, const uint8_t* pool, int64_t n_items,
                             const orc_ingest_item* items, const int32_t* block_table,
                             int64_t bt_stride, int64_t num_pages, uint8_t* arena, int64_t layer_lo,
                             int64_t layer_hi, int threads, int layout, int64_t arena_layer0) {
  const int64_t L = s->layers, H = s->kv_heads, D = s->head_dim, E = s->dtype_bytes;
  const int64_t C = s->chunk_tokens, P = s->page_tokens;
  const int64_t Hl = H / s->tp_size, h0 = s->tp_rank * Hl;
  const int64_t ppc = C / P;
  const int64_t row = H * D * E, run = Hl * D * E;
  const int64_t chunk_bytes = L * 2 * C * row;
  const int64_t n_work = n_items * (layer_hi - layer_lo);
  (void)threads;
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads > 0 ? threads : 1)
  for (int64_t w = 0; w < n_work; ++w) {
    const orc_ingest_item it = items[w / (layer_hi - layer_lo)];
    const int64_t l = layer_lo + w % (layer_hi - layer_lo);
    const uint8_t* chunk = pool + it.src_slot * chunk_bytes;
    for (int64_t kv = 0; kv < 2; ++kv) {
      for (int64_t j = 0; j < ppc; ++j) {
        const int64_t page = block_table[it.bt_row * bt_stride + it.chunk_index * ppc + j];
        const int64_t seg = P * run; /* one (layer, K|V, page) unit */
        uint8_t* dst = arena + (l - arena_layer0) * 2 * num_pages * seg +
                       (layout == 0 ? (kv * num_pages + page) * seg : (page * 2 + kv) * seg);
        const uint8_t* src = chunk + ((l * 2 + kv) * C + j * P) * row + h0 * D * E;
        if (layout == 2) { /* [Hl][P][D]: head h's row of token t */
          for (int64_t h = 0; h < Hl; ++h)
            for (int64_t t = 0; t < P; ++t)
              memcpy(dst + (h * P + t) * D * E, src + t * row + h * D * E, (size_t)(D * E));
        } else if (run == row) {
          memcpy(dst, src, (size_t)(P * row));
        } else {
          for (int64_t t = 0; t < P; ++t) memcpy(dst + t * run, src + t * row, (size_t)run);
        }
      }
    }
  }
}

void orc_scatter_ref_layout(const orc_kv_shape* s, const uint8_t* pool, int64_t n_items,
                            const orc_ingest_item* items, const int32_t* block_table,
                            int64_t bt_stride, int64_t num_pages, uint8_t* arena, int64_t layer_lo,
                            int64_t layer_hi, int threads, int layout) {
  scatter_ref_impl(s, pool, n_items, items, block_table, bt_stride, num_pages, arena, layer_lo,
                   layer_hi, threads, layout, 0);
}

/* Layers [layer_lo, layer_hi) only, into an arena buffer holding just those layers (full-size
 * parity checks of sampled layers without a whole-model host arena). */
void orc_scatter_ref_window(const orc_kv_shape* s, const uint8_t* pool, int64_t n_items,
                            const orc_ingest_item* items, const int32_t* block_table,
                            int64_t bt_stride, int64_t num_pages, uint8_t* arena_window,
                            int64_t layer_lo, int64_t layer_hi, int threads, int layout) {
  scatter_ref_impl(s, pool, n_items, items, block_table, bt_stride, num_pages, arena_window,
                   layer_lo, layer_hi, threads, layout, layer_lo);
}

void orc_scatter_ref(const orc_kv_shape* s, const uint8_t* pool, int64_t n_items,
                     const orc_ingest_item* items, const int32_t* block_table,
                     int64_t bt_stride, int64_t num_pages, uint8_t* arena, int64_t layer_lo,
                     int64_t layer_hi, int threads) {
  orc_scatter_ref_layout(s, pool, n_items, items, block_table, bt_stride, num_pages, arena, layer_lo,
                         layer_hi, threads, 0);
}

/* ------------------------------------------------------------------------ */
/* synthetic data: counter-based, identical on CPU and GPU                    */
/* ------------------------------------------------------------------------ */

/* splitmix64 finaliser */
uint64_t orc_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* 8-byte word `word_index` of the synthetic pool: four bf16 values with the top
 * exponent bit cleared, so every value is finite. */
uint64_t orc_synth_word(uint64_t seed, uint64_t word_index) {
  return orc_mix64(seed ^ (word_index * 0xd1b54a32d192ed03ull)) & 0xbfffbfffbfffbfffull;
}

void orc_synth_fill(uint64_t seed, uint64_t first_word, uint64_t n_words, uint64_t* out,
                    int threads) {
  (void)threads;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
  for (int64_t i = 0; i < (int64_t)n_words; ++i)
    out[i] = orc_synth_word(seed, first_word + (uint64_t)i);
}

/* Token id of `stream` at position `pos` (17-bit ids).  Requests whose prefix comes from
 * the same document share `stream` for their first shared_len tokens. */
uint32_t orc_token_id(uint64_t seed, uint64_t stream, uint64_t pos) {
  return (uint32_t)(orc_mix64(seed + stream * 0x9e3779b97f4a7c15ull +
                              pos * 0xd1b54a32d192ed03ull) >> 47);
}

void orc_gen_tokens(uint64_t seed, int64_t n_req, const int64_t* offsets, const int64_t* doc,
                    const int64_t* shared_len, int32_t* out, int threads) {
  (void)threads;
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads > 0 ? threads : 1)
  for (int64_t r = 0; r < n_req; ++r) {
    const int64_t n = offsets[r + 1] - offsets[r];
    for (int64_t p = 0; p < n; ++p) {
      const uint64_t stream = p < shared_len[r] ? (uint64_t)doc[r] : (1ull << 40) + (uint64_t)r;
      out[offsets[r] + p] = (int32_t)orc_token_id(seed, stream, (uint64_t)p);
    }
  }
}

/* ------------------------------------------------------------------------ */
/* prefix chunk hash.  The reference's only hash is byte-wise FNV-1a-64       */
/* (engine.cpp:500-507, seeded with 0xcbf29ce484222325 at :518); it has no     */
/* prefix hasher.  Definition (frozen here, GPU must match): */
/*   step(h, w)  = (h ^ w) * FNV_PRIME           (FNV-1a on a 64-bit word)     */
/*   word k      = u32 tok[2k] | u32 tok[2k+1] << 32 (the little-endian 8-byte  */
/*                 image of two consecutive int32 token ids)                   */
/*   leaf j      = fold step, from FNV_OFFSET, over the 8 words                   */
/*                 32k + 2j, 32k + 2j + 1 for k = 0..3 (j = 0..15): the words a */
/*                 16-lane group reads with four fully coalesced 16-byte loads  */
/*   pair(a, b)  = step(step(FNV_OFFSET, a), b)                                 */
/*   digest      = 4-level pairwise tree of pair() over the 16 leaves, in order */
/*   H_c         = pair(H_{c-1}, digest_c),  H_{-1} = rotl(FNV_OFFSET, 32)       */
/* Only full 256-token chunks are hashed (floor rule, types.cpp:73-79).        */
/* ------------------------------------------------------------------------ */

/* byte-wise FNV-1a, engine.cpp:500-507 */
uint64_t orc_fnv1a_bytes(uint64_t h, const void* data, size_t len) {
  const unsigned char* b = (const unsigned char*)data;
  for (size_t i = 0; i < len; ++i) {
    h ^= b[i];
    h *= FNV_PRIME;
  }
  return h;
}

static inline uint64_t step(uint64_t h, uint64_t w) { return (h ^ w) * FNV_PRIME; }
static inline uint64_t pair(uint64_t a, uint64_t b) { return step(step(FNV_OFFSET, a), b); }

uint64_t orc_chunk_digest(const int32_t* tok) {
  uint64_t node[16];
  for (int j = 0; j < 16; ++j) {
    uint64_t h = FNV_OFFSET;
    for (int k = 0; k < 4; ++k) {
      for (int e = 0; e < 2; ++e) {
        const int t = 2 * (32 * k + 2 * j + e); /* first token of word 32k + 2j + e */
        h = step(h, (uint64_t)(uint32_t)tok[t] | ((uint64_t)(uint32_t)tok[t + 1] << 32));
      }
    }
    node[j] = h;
  }
  for (int width = 8; width >= 1; width /= 2)
    for (int i = 0; i < width; ++i) node[i] = pair(node[2 * i], node[2 * i + 1]);
  return node[0];
}

uint64_t orc_chain(uint64_t prev, uint64_t digest) { return pair(prev, digest); }

/* Writes the chained hash of every full chunk of every request; request r's chunk
 * hashes start at chunk_offsets[r] (chunk_offsets[r+1]-chunk_offsets[r] = floor(len/256)).
 * Returns the total number of chunk hashes. */
int64_t orc_hash_prefix_chunks(int64_t n_req, const int64_t* offsets, const int32_t* tokens,
                               const int64_t* chunk_offsets, uint64_t* out, int threads) {
  (void)threads;
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads > 0 ? threads : 1)
  for (int64_t r = 0; r < n_req; ++r) {
    const int64_t nchunks = (offsets[r + 1] - offsets[r]) / 256;
    uint64_t h = (FNV_OFFSET << 32) | (FNV_OFFSET >> 32);
    for (int64_t c = 0; c < nchunks; ++c) {
      h = orc_chain(h, orc_chunk_digest(tokens + offsets[r] + c * 256));
      out[chunk_offsets[r] + c] = h;
    }
  }
  return n_req > 0 ? chunk_offsets[n_req] : 0;
}
