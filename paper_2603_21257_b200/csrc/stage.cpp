// stage.cpp — the real-time L2->L1 load stage (tsb_stage_*).
//
// SimEngine's dispatch rules with real bytes and real time (reference: core/src/engine.cpp):
//   * pick order: the batched GPU scorer (K4/K5) orders the batch by PriorityKey under the chosen
//     policy -- the order best_pending()/admit() would produce for a queue present at one instant
//     (engine.cpp:306-312, 341-355; keys ignore `now`, scheduler.cpp:47);
//   * admission reserves L1 for every planned chunk in block order (proactive allocation,
//     engine.cpp:419) through the TierLedger-semantics paged allocator; reservations that do not
//     fit wait FIFO and are granted by later releases (engine.cpp:38-49, 388-397);
//   * a chunk is ingested only once its pages are granted (grant-before-hop, engine.cpp:434-436),
//     requests are served in pick order (pcie_dispatch scans admitted_ in pick order, :427-446);
//   * a request's L1 pages are released when its prefill completes (ComputeDone, :280-282); with
//     prefill disabled, when its last layer is resident.
// The simulator's event queue and clock are replaced by CUDA streams and events: ingest on the
// caller's stream, synthetic prefill (K6) on a lower-priority compute stream that waits on the
// request's per-layer fences, and the host thread blocks on the oldest request only when the
// ledger has deferred reservations and nothing else can be dispatched.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <ctime>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "kernels.h"

using tsb::fail;

namespace {

struct ReqRt {
  int64_t q_index = 0;
  int64_t id = 0;
  int64_t n_chunks = 0;
  int64_t compute_tokens = 0;
  const int64_t* slots = nullptr;
  int32_t row = -1;
  std::vector<int32_t> ready;  // granted, not yet ingested (block order)
  int64_t issued = 0;
  int32_t deferred = 0;
  bool finished_issue = false;
  bool released = false;
  cudaEvent_t ev_first = nullptr, ev_resident = nullptr, ev_done = nullptr;
};

double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

}  // namespace

struct tsb_stage {
  tsb_l1* l1 = nullptr;
  tsb_pool* pool = nullptr;
  tsb_pool* hbm_pool = nullptr;  // HBM tier: slots < 0 name slot ~slot of this pool
  tsb_kv_shape shape{};
  int device = 0;
  tsb_scorer* scorer = nullptr;
  cudaStream_t compute = nullptr;
  std::vector<cudaEvent_t> timing_pool;  // 3 per request, grown on demand
  std::vector<cudaEvent_t> layer_ev;     // per-layer fences (reused across requests)
  cudaEvent_t ev_start = nullptr;
  std::vector<cudaEvent_t> call_ev;      // per ingest call (trace only)
  std::vector<tsb_trace_row> trace;
  uint64_t seq = 0;
};

extern "C" {

tsb_status tsb_stage_create(tsb_l1* l1, tsb_pool* pool, tsb_stage** out) {
  auto* s = new tsb_stage();
  s->l1 = l1;
  s->pool = pool;
  TSB_TRY(tsb_l1_shape(l1, &s->shape));
  s->device = tsb_l1_device(l1);
  TSB_CUDA_TRY(cudaSetDevice(s->device));
  int lo = 0, hi = 0;
  TSB_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  // Prefill gets the LOWEST priority so the ingest scatter kernels interleave ahead of it.
  TSB_CUDA_TRY(cudaStreamCreateWithPriority(&s->compute, cudaStreamNonBlocking, lo));
  TSB_CUDA_TRY(cudaEventCreate(&s->ev_start));
  s->layer_ev.resize(static_cast<size_t>(s->shape.layers));
  for (auto& e : s->layer_ev) TSB_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  TSB_TRY(tsb_scorer_create(s->device, 1024, &s->scorer));
  *out = s;
  return TSB_OK;
}

tsb_status tsb_stage_set_hbm_tier(tsb_stage* s, tsb_pool* hbm_pool) {
  if (hbm_pool && tsb_pool_chunk_bytes(hbm_pool) != tsb_pool_chunk_bytes(s->pool))
    return fail(TSB_VALIDATION, "stage: the HBM tier's chunk geometry differs from the L2 pool's");
  s->hbm_pool = hbm_pool;
  return TSB_OK;
}

void tsb_stage_destroy(tsb_stage* s) {
  if (!s) return;
  for (auto e : s->timing_pool) cudaEventDestroy(e);
  for (auto e : s->layer_ev) cudaEventDestroy(e);
  for (auto e : s->call_ev) cudaEventDestroy(e);
  if (s->ev_start) cudaEventDestroy(s->ev_start);
  if (s->compute) cudaStreamDestroy(s->compute);
  tsb_scorer_destroy(s->scorer);
  delete s;
}

tsb_status tsb_stage_trace(tsb_stage* s, tsb_trace_row* out, int64_t cap, int64_t* n) {
  *n = static_cast<int64_t>(s->trace.size());
  for (int64_t i = 0; i < *n && i < cap; ++i) out[i] = s->trace[i];
  return TSB_OK;
}

tsb_status tsb_stage_run(tsb_stage* s, int64_t n, const tsb_queue* q, const tsb_cluster* c,
                         const double models[4], const int64_t* slot_offsets,
                         const int64_t* slots, const tsb_stage_options* opt, void* stream,
                         tsb_stage_request* results, tsb_stage_stats* stats) {
  const double wall0 = now_s();
  const uint64_t launches0 = tsb_kernel_launch_count();
  auto st = static_cast<cudaStream_t>(stream);
  const int64_t L = s->shape.layers;
  int64_t chunk_bytes_full = 0, page_bytes = 0, chunk_bytes = 0;
  TSB_TRY(tsb_kv_shape_info(&s->shape, &chunk_bytes_full, &page_bytes, &chunk_bytes));
  TSB_TRY(tsb_cluster_validate(c));
  if (c->block_size_tokens != s->shape.chunk_tokens)
    return fail(TSB_VALIDATION, "stage: cluster block_size_tokens must equal the KV chunk_tokens");
  s->trace.clear();
  s->seq = 0;
  auto row = [&](double t, int kind, int stg, int tier, int64_t rid, int32_t blk, int64_t bytes) {
    if (opt->record_trace) s->trace.push_back({t, s->seq++, kind, stg, tier, blk, rid, bytes});
  };

  // ---- plans (types.cpp:85-101) and capacity check (engine.cpp:213-217) ----------------------
  std::vector<ReqRt> reqs(static_cast<size_t>(n));
  std::unordered_map<int64_t, size_t> by_id;
  const int64_t l1_capacity = tsb_l1_capacity(s->l1);
  for (int64_t i = 0; i < n; ++i) {
    int64_t cached = 0, compute = 0, nb = 0, bt = 0, bb = 0;
    TSB_TRY(tsb_derive_block_plan(q, i, c, &cached, &compute, &nb, &bt, &bb));
    ReqRt& r = reqs[i];
    r.q_index = i;
    r.id = q->id[i];
    r.n_chunks = nb;
    r.compute_tokens = compute;
    r.slots = slots + slot_offsets[i];
    if (slot_offsets[i + 1] - slot_offsets[i] != nb)
      return fail(TSB_VALIDATION, "stage: request " + std::to_string(r.id) + " lists " +
                                      std::to_string(slot_offsets[i + 1] - slot_offsets[i]) +
                                      " pool slots for a plan of " + std::to_string(nb) + " chunks");
    for (int64_t k = 0; k < nb; ++k) {
      const int64_t sl = r.slots[k];
      const bool ok = sl >= 0 ? sl < tsb_pool_slots(s->pool)
                              : (s->hbm_pool && ~sl < tsb_pool_slots(s->hbm_pool));
      if (!ok) return fail(TSB_VALIDATION, "stage: pool slot out of range");
    }
    if (nb * chunk_bytes > l1_capacity)
      return fail(TSB_CAPACITY, "request " + std::to_string(r.id) + ": " +
                                    std::to_string(nb * chunk_bytes) +
                                    " resident bytes can never fit");
    if (!by_id.emplace(r.id, static_cast<size_t>(i)).second)
      return fail(TSB_VALIDATION, "run_simulation: duplicate request id " + std::to_string(r.id));
  }
  while (s->timing_pool.size() < static_cast<size_t>(3 * n)) {
    cudaEvent_t e;
    TSB_CUDA_TRY(cudaEventCreate(&e));
    s->timing_pool.push_back(e);
  }
  for (int64_t i = 0; i < n; ++i) {
    reqs[i].ev_first = s->timing_pool[3 * i];
    reqs[i].ev_resident = s->timing_pool[3 * i + 1];
    reqs[i].ev_done = s->timing_pool[3 * i + 2];
  }

  // ---- pick order (K4 + K5 on the GPU) ----------------------------------------------------------
  std::vector<int64_t> order(static_cast<size_t>(n));
  if (n > 0)
    TSB_TRY(tsb_score_queue(s->scorer, stream, n, q, opt->policy, models, c, nullptr, nullptr,
                            nullptr, order.data()));
  std::vector<int64_t> pos_of(static_cast<size_t>(n));
  for (int64_t k = 0; k < n; ++k) pos_of[order[k]] = k;

  TSB_CUDA_TRY(cudaEventRecord(s->ev_start, st));
  const double host0 = now_s();
  const int ctas = opt->prefill_ctas > 0 ? opt->prefill_ctas : 148;
  int64_t ingest_calls = 0, deferred_total = 0, releases = 0, bytes_total = 0;
  uint64_t verify_mismatches = 0;

  auto finish_request_events = [&](ReqRt& r) -> tsb_status {
    // Called once the request's last chunk has been dispatched: ev_first / ev_resident were
    // recorded by that ingest call (or here for an empty plan); now the prefill and ev_done.
    if (r.n_chunks == 0) {
      TSB_CUDA_TRY(cudaEventRecord(r.ev_first, st));
      TSB_CUDA_TRY(cudaEventRecord(r.ev_resident, st));
      for (int64_t l = 0; l < L; ++l) TSB_CUDA_TRY(cudaEventRecord(s->layer_ev[l], st));
    }
    if (opt->prefill) {
      const double ct = static_cast<double>(r.compute_tokens);
      const double secs = c->compute_base + c->compute_per_token * ct + c->compute_quadratic * ct * ct;
      const auto per_layer_ns = static_cast<uint64_t>(secs * 1e9 / static_cast<double>(L));
      for (int64_t l = 0; l < L; ++l) {
        cudaEvent_t fence = r.ev_resident;
        if (opt->layer_events) fence = l == 0 ? r.ev_first : l == L - 1 ? r.ev_resident : s->layer_ev[l];
        TSB_CUDA_TRY(cudaStreamWaitEvent(s->compute, fence, 0));
        for (uint64_t done = 0; done < per_layer_ns; done += 250000)
          TSB_CUDA_TRY(tsb::launch_prefill_burn(std::min<uint64_t>(250000, per_layer_ns - done),
                                                ctas, nullptr, s->compute));
      }
      TSB_CUDA_TRY(cudaEventRecord(r.ev_done, s->compute));
    } else {
      TSB_CUDA_TRY(cudaEventRecord(r.ev_done, st));
    }
    r.finished_issue = true;
    return TSB_OK;
  };

  // pcie_dispatch (engine.cpp:427-446): serve granted chunks of admitted requests in pick order.
  auto dispatch = [&]() -> tsb_status {
    bool synced = false;
    for (int64_t k = 0; k < n; ++k) {
      ReqRt& r = reqs[order[k]];
      if (r.finished_issue || r.ready.empty()) continue;
      if (!synced) {
        TSB_TRY(tsb_l1_sync_block_table(s->l1, stream));
        synced = true;
      }
      std::vector<tsb_ingest_item> items;
      items.reserve(r.ready.size());
      for (int32_t ch : r.ready) {
        items.push_back(tsb_ingest_item{r.slots[ch], r.row, ch});
        row(now_s() - host0, 4, 1, -1, r.id, ch, chunk_bytes);  // DispatchWake(Pcie)
      }
      r.issued += static_cast<int64_t>(items.size());
      r.ready.clear();
      const bool last = r.issued == r.n_chunks;
      std::vector<void*> evs;
      void* const* evp = nullptr;
      if (last) {
        // Timing events double as the layer-0 and last-layer fences.
        evs.assign(static_cast<size_t>(L), nullptr);
        if (opt->layer_events)
          for (int64_t l = 1; l + 1 < L; ++l) evs[l] = s->layer_ev[l];
        evs[0] = r.ev_first;
        evs[L - 1] = r.ev_resident;
        evp = evs.data();
      }
      TSB_TRY(tsb_ingest_tiered(s->l1, s->pool, s->hbm_pool, items.data(),
                                static_cast<int64_t>(items.size()), 0, L, opt->mode, stream, evp));
      if (last && L == 1) TSB_CUDA_TRY(cudaEventRecord(r.ev_first, st));
      if (opt->record_trace) {
        cudaEvent_t ce;
        TSB_CUDA_TRY(cudaEventCreate(&ce));
        TSB_CUDA_TRY(cudaEventRecord(ce, st));
        s->call_ev.push_back(ce);
        for (const auto& it : items)  // TransferDone(Pcie); time filled in after the run
          row(-static_cast<double>(s->call_ev.size()), 1, 1, -1, r.id, it.chunk_index, chunk_bytes);
      }
      ++ingest_calls;
      bytes_total += static_cast<int64_t>(items.size()) * chunk_bytes;
      if (last) TSB_TRY(finish_request_events(r));
    }
    return TSB_OK;
  };

  // admit (engine.cpp:341-355) in pick order: reserve L1 for every planned chunk.
  int64_t total_chunks = 0;
  for (const auto& r : reqs) total_chunks += r.n_chunks;
  std::vector<tsb_grant> grants(static_cast<size_t>(std::max<int64_t>(total_chunks, 1)));
  for (int64_t k = 0; k < n; ++k) {
    ReqRt& r = reqs[order[k]];
    for (int64_t ch = 0; ch < r.n_chunks; ++ch) {
      int granted = 0;
      TSB_TRY(tsb_l1_request(s->l1, r.id, static_cast<int32_t>(ch), chunk_bytes, &granted, &r.row));
      if (granted) {
        r.ready.push_back(static_cast<int32_t>(ch));
        row(now_s() - host0, 2, -1, 2, r.id, static_cast<int32_t>(ch), chunk_bytes);
      } else {
        ++r.deferred;
        ++deferred_total;
      }
    }
    if (r.n_chunks == 0) TSB_TRY(finish_request_events(r));
  }
  TSB_TRY(dispatch());

  // Complete requests in pick order; each release may grant deferred reservations (FIFO), whose
  // chunks are dispatched right away so the link never idles while the host waits.
  for (int64_t k = 0; k < n; ++k) {
    ReqRt& r = reqs[order[k]];
    if (!r.finished_issue)
      return fail(TSB_CAPACITY, "stage: request " + std::to_string(r.id) +
                                    " is blocked on L1 pages held by later requests");
    TSB_CUDA_TRY(cudaEventSynchronize(r.ev_done));
    if (opt->verify_seed && r.n_chunks > 0) {
      std::vector<tsb_ingest_item> items;
      // both tiers hold the synthetic pattern of the seed at their own slot index
      for (int64_t ch = 0; ch < r.n_chunks; ++ch)
        items.push_back(tsb_ingest_item{r.slots[ch] < 0 ? ~r.slots[ch] : r.slots[ch], r.row,
                                        static_cast<int32_t>(ch)});
      uint64_t mm = 0;
      TSB_TRY(tsb_l1_verify_synthetic(s->l1, items.data(), r.n_chunks, 0, L, opt->verify_seed,
                                      tsb_pool_chunk_bytes(s->pool), stream, &mm));
      verify_mismatches += mm;
    }
    // ComputeDone (engine.cpp:349-358): bytes = compute_tokens * bytes_per_token, then release.
    row(now_s() - host0, 3, 2, -1, r.id, -1, r.compute_tokens * c->bytes_per_token);
    if (r.row >= 0) {
      int64_t ng = 0;
      TSB_TRY(tsb_l1_release_request(s->l1, r.id, grants.data(),
                                     static_cast<int64_t>(grants.size()), &ng));
      ++releases;
      const double t = now_s() - host0;
      for (int64_t g = 0; g < ng; ++g) {
        ReqRt& w = reqs[by_id.at(grants[g].request_id)];
        w.ready.push_back(grants[g].block_index);
        row(t, 2, -1, 2, w.id, grants[g].block_index, grants[g].bytes);
      }
      TSB_TRY(dispatch());
    }
    r.released = true;
  }
  TSB_CUDA_TRY(cudaStreamSynchronize(st));

  // ---- results --------------------------------------------------------------------------------
  float last_ms = 0.f;
  for (int64_t i = 0; i < n; ++i) {
    ReqRt& r = reqs[i];
    float a = 0.f, b = 0.f, d = 0.f;
    TSB_CUDA_TRY(cudaEventElapsedTime(&a, s->ev_start, r.ev_first));
    TSB_CUDA_TRY(cudaEventElapsedTime(&b, s->ev_start, r.ev_resident));
    TSB_CUDA_TRY(cudaEventElapsedTime(&d, s->ev_start, r.ev_done));
    last_ms = std::max(last_ms, b);
    if (results)
      results[i] = tsb_stage_request{r.id, static_cast<int32_t>(pos_of[i]), r.deferred, r.n_chunks,
                                     r.n_chunks * chunk_bytes, a, b, d, 0.0, 0.0};
  }
  if (opt->record_trace) {
    for (auto& tr : s->trace) {
      if (tr.time < 0) {
        float ms = 0.f;
        TSB_CUDA_TRY(cudaEventElapsedTime(&ms, s->ev_start, s->call_ev[static_cast<size_t>(-tr.time) - 1]));
        tr.time = ms * 1e-3;
      }
    }
    for (auto e : s->call_ev) cudaEventDestroy(e);
    s->call_ev.clear();
  }
  if (stats) {
    stats->bytes = bytes_total;
    stats->device_ms = last_ms;
    stats->wall_ms = (now_s() - wall0) * 1e3;
    stats->ingest_calls = ingest_calls;
    stats->deferred_chunks = deferred_total;
    stats->releases = releases;
    stats->kernel_launches = static_cast<int64_t>(tsb_kernel_launch_count() - launches0);
    stats->verify_mismatches = verify_mismatches;
  }
  return TSB_OK;
}

tsb_status tsb_stage_run_online(tsb_stage* s, int64_t n, const tsb_queue* q,
                                const tsb_cluster* c, const double models[4],
                                const int64_t* slot_offsets, const int64_t* slots,
                                const tsb_stage_options* opt, void* stream,
                                tsb_stage_request* results, tsb_stage_stats* stats) {
  const double wall0 = now_s();
  const uint64_t launches0 = tsb_kernel_launch_count();
  auto st = static_cast<cudaStream_t>(stream);
  const int64_t L = s->shape.layers;
  int64_t chunk_bytes_full = 0, page_bytes = 0, chunk_bytes = 0;
  TSB_TRY(tsb_kv_shape_info(&s->shape, &chunk_bytes_full, &page_bytes, &chunk_bytes));
  TSB_TRY(tsb_cluster_validate(c));
  if (c->block_size_tokens != s->shape.chunk_tokens)
    return fail(TSB_VALIDATION, "stage: cluster block_size_tokens must equal the KV chunk_tokens");
  if (n == 0) return TSB_OK;
  struct Rt {
    int64_t id = 0, n_chunks = 0, compute_tokens = 0;
    const int64_t* slots = nullptr;
    int32_t row = -1, deferred = 0;
    std::vector<int32_t> ready;
    int64_t issued = 0, granted = 0;
    bool arrived = false, admitted = false, dispatched_all = false, resident = false,
         started = false, finished = false;
    double arrival = 0.0, admit_t = 0.0;
    cudaEvent_t ev_first = nullptr, ev_resident = nullptr, ev_done = nullptr;
  };
  std::vector<Rt> R(static_cast<size_t>(n));
  std::unordered_map<int64_t, size_t> by_id;
  const int64_t l1_capacity = tsb_l1_capacity(s->l1);
  double first_arrival = q->arrival[0];
  for (int64_t i = 0; i < n; ++i) first_arrival = std::min(first_arrival, q->arrival[i]);
  for (int64_t i = 0; i < n; ++i) {
    int64_t cached = 0, compute = 0, nb = 0, bt = 0, bb = 0;
    TSB_TRY(tsb_derive_block_plan(q, i, c, &cached, &compute, &nb, &bt, &bb));
    Rt& r = R[i];
    r.id = q->id[i];
    r.n_chunks = nb;
    r.compute_tokens = compute;
    r.slots = slots + slot_offsets[i];
    r.arrival = q->arrival[i] - first_arrival;
    if (slot_offsets[i + 1] - slot_offsets[i] != nb)
      return fail(TSB_VALIDATION, "stage: request " + std::to_string(r.id) + " lists " +
                                      std::to_string(slot_offsets[i + 1] - slot_offsets[i]) +
                                      " pool slots for a plan of " + std::to_string(nb) + " chunks");
    if (nb * chunk_bytes > l1_capacity)
      return fail(TSB_CAPACITY, "request " + std::to_string(r.id) + ": " +
                                    std::to_string(nb * chunk_bytes) +
                                    " resident bytes can never fit");
    if (!by_id.emplace(r.id, static_cast<size_t>(i)).second)
      return fail(TSB_VALIDATION, "run_simulation: duplicate request id " + std::to_string(r.id));
  }
  while (s->timing_pool.size() < static_cast<size_t>(3 * n)) {
    cudaEvent_t e;
    TSB_CUDA_TRY(cudaEventCreate(&e));
    s->timing_pool.push_back(e);
  }
  for (int64_t i = 0; i < n; ++i) {
    R[i].ev_first = s->timing_pool[3 * i];
    R[i].ev_resident = s->timing_pool[3 * i + 1];
    R[i].ev_done = s->timing_pool[3 * i + 2];
  }
  // Priority keys from the GPU scorer (K4), compared with PriorityKey::operator< on the host.
  std::vector<double> primary(static_cast<size_t>(n));
  std::vector<int64_t> order(static_cast<size_t>(n));
  TSB_TRY(tsb_score_queue(s->scorer, stream, n, q, opt->policy, models, c, nullptr, nullptr,
                          primary.data(), order.data()));
  auto key_less = [&](size_t a, size_t b) {
    if (primary[a] != primary[b]) return primary[a] < primary[b];
    if (q->arrival[a] != q->arrival[b]) return q->arrival[a] < q->arrival[b];
    return q->id[a] < q->id[b];
  };
  std::vector<size_t> by_arrival(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) by_arrival[i] = static_cast<size_t>(i);
  std::stable_sort(by_arrival.begin(), by_arrival.end(),
                   [&](size_t a, size_t b) { return R[a].arrival < R[b].arrival; });

  cudaEvent_t ev_ingest = nullptr, ev_compute = nullptr;
  TSB_CUDA_TRY(cudaEventCreateWithFlags(&ev_ingest, cudaEventDisableTiming));
  TSB_CUDA_TRY(cudaEventCreateWithFlags(&ev_compute, cudaEventDisableTiming));
  bool ingest_issued = false, compute_issued = false;
  const int ctas = opt->prefill_ctas > 0 ? opt->prefill_ctas : 148;
  std::vector<tsb_grant> grants(4096);
  int64_t ingest_calls = 0, deferred_total = 0, releases = 0, bytes_total = 0;
  uint64_t verify_mismatches = 0;
  std::vector<size_t> pending, admitted;
  size_t next_arrival = 0, finished = 0;
  int64_t pick = 0;
  std::vector<int32_t> pick_pos(static_cast<size_t>(n), -1);

  TSB_CUDA_TRY(cudaEventRecord(s->ev_start, st));
  const double host0 = now_s();
  auto done = [](cudaEvent_t e) { return cudaEventQuery(e) == cudaSuccess; };
  tsb_status status = TSB_OK;
  auto fail_out = [&](tsb_status st_) {
    status = st_;
    return st_;
  };

  while (finished < static_cast<size_t>(n)) {
    const double now = now_s() - host0;
    while (next_arrival < by_arrival.size() && R[by_arrival[next_arrival]].arrival <= now) {
      R[by_arrival[next_arrival]].arrived = true;
      pending.push_back(by_arrival[next_arrival++]);
    }
    bool progress = true;
    while (progress) {
      progress = false;
      // ComputeDone -> release this request's L1 pages; FIFO grants to waiting reservations.
      for (size_t i : admitted) {
        Rt& r = R[i];
        if (!r.started || r.finished || !done(r.ev_done)) continue;
        r.finished = true;
        ++finished;
        progress = true;
        if (opt->verify_seed && r.n_chunks > 0) {  // opt-in check (synchronises the stream)
          std::vector<tsb_ingest_item> items;
          for (int64_t ch = 0; ch < r.n_chunks; ++ch)
            items.push_back(tsb_ingest_item{r.slots[ch] < 0 ? ~r.slots[ch] : r.slots[ch], r.row,
                                            static_cast<int32_t>(ch)});
          uint64_t mm = 0;
          if (tsb_l1_verify_synthetic(s->l1, items.data(), r.n_chunks, 0, L, opt->verify_seed,
                                      tsb_pool_chunk_bytes(s->pool), stream, &mm) != TSB_OK)
            return fail_out(TSB_CUDA);
          verify_mismatches += mm;
        }
        if (r.row >= 0) {
          int64_t ng = 0;
          if (grants.size() < static_cast<size_t>(tsb_l1_deferred(s->l1)) + 1)
            grants.resize(static_cast<size_t>(tsb_l1_deferred(s->l1)) + 1);
          if (tsb_l1_release_request(s->l1, r.id, grants.data(),
                                     static_cast<int64_t>(grants.size()), &ng) != TSB_OK)
            return fail_out(TSB_VALIDATION);
          ++releases;
          for (int64_t g = 0; g < ng; ++g) {
            Rt& w = R[by_id.at(grants[g].request_id)];
            w.ready.push_back(grants[g].block_index);
            ++w.granted;
          }
        }
      }
      // PcieDone of a request's last chunk -> L1 resident -> compute ready.
      for (size_t i : admitted) {
        Rt& r = R[i];
        if (r.dispatched_all && !r.resident && done(r.ev_resident)) {
          r.resident = true;
          progress = true;
        }
      }
      // try_admit, decoupled (engine.cpp:318-339): the first stage must be idle with no backlog.
      if (!pending.empty()) {
        size_t bi = 0;
        for (size_t k = 1; k < pending.size(); ++k)
          if (key_less(pending[k], pending[bi])) bi = k;
        Rt& r = R[pending[bi]];
        bool backlog = false;
        for (size_t i : admitted)
          if (!R[i].dispatched_all) backlog = true;
        bool can = false;
        if (r.n_chunks > 0) {
          can = !backlog && (!ingest_issued || done(ev_ingest));
        } else {
          bool ready_waiting = false;
          for (size_t i : admitted)
            if (R[i].resident && !R[i].started) ready_waiting = true;
          can = (!compute_issued || done(ev_compute)) && !ready_waiting;
        }
        if (can) {
          const size_t idx = pending[bi];
          pending.erase(pending.begin() + static_cast<std::ptrdiff_t>(bi));
          r.admitted = true;
          r.admit_t = now_s() - host0;
          pick_pos[idx] = static_cast<int32_t>(pick++);
          admitted.push_back(idx);
          for (int64_t ch = 0; ch < r.n_chunks; ++ch) {
            int granted = 0;
            const tsb_status rs = tsb_l1_request(s->l1, r.id, static_cast<int32_t>(ch), chunk_bytes,
                                                 &granted, &r.row);
            if (rs != TSB_OK) return fail_out(rs);
            if (granted) {
              r.ready.push_back(static_cast<int32_t>(ch));
              ++r.granted;
            } else {
              ++r.deferred;
              ++deferred_total;
            }
          }
          if (r.n_chunks == 0) {
            r.dispatched_all = true;
            cudaEventRecord(r.ev_first, st);
            cudaEventRecord(r.ev_resident, st);
          }
          progress = true;
        }
      }
      // pcie_dispatch: granted chunks of admitted requests, in admission order.
      for (size_t i : admitted) {
        Rt& r = R[i];
        if (r.ready.empty()) continue;
        if (tsb_l1_sync_block_table(s->l1, stream) != TSB_OK) return fail_out(TSB_CUDA);
        std::vector<tsb_ingest_item> items;
        for (int32_t ch : r.ready) items.push_back(tsb_ingest_item{r.slots[ch], r.row, ch});
        r.ready.clear();
        r.issued += static_cast<int64_t>(items.size());
        const bool last = r.issued == r.n_chunks;
        std::vector<void*> evs;
        if (last) {
          evs.assign(static_cast<size_t>(L), nullptr);
          evs[0] = r.ev_first;
          evs[L - 1] = r.ev_resident;
        }
        const tsb_status is = tsb_ingest_tiered(s->l1, s->pool, s->hbm_pool, items.data(),
                                                static_cast<int64_t>(items.size()), 0, L,
                                                opt->mode, stream, last ? evs.data() : nullptr);
        if (is != TSB_OK) return fail_out(is);
        if (last && L == 1) cudaEventRecord(r.ev_first, st);
        cudaEventRecord(ev_ingest, st);
        ingest_issued = true;
        ++ingest_calls;
        bytes_total += static_cast<int64_t>(items.size()) * chunk_bytes;
        if (last) r.dispatched_all = true;
        progress = true;
      }
      // try_start_compute (engine.cpp:448-473): best key among resident, not started.
      if (!compute_issued || done(ev_compute)) {
        size_t best = SIZE_MAX;
        for (size_t i : admitted) {
          const Rt& r = R[i];
          if (!r.resident || r.started) continue;
          if (best == SIZE_MAX || key_less(i, best)) best = i;
        }
        if (best != SIZE_MAX) {
          Rt& r = R[best];
          r.started = true;
          const double ct = static_cast<double>(r.compute_tokens);
          const double secs =
              c->compute_base + c->compute_per_token * ct + c->compute_quadratic * ct * ct;
          const auto ns = static_cast<uint64_t>(secs * 1e9);
          cudaStreamWaitEvent(s->compute, r.ev_resident, 0);
          for (uint64_t t = 0; t < ns; t += 250000)
            if (tsb::launch_prefill_burn(std::min<uint64_t>(250000, ns - t), ctas, nullptr,
                                         s->compute) != cudaSuccess)
              return fail_out(TSB_CUDA);
          cudaEventRecord(r.ev_done, s->compute);
          cudaEventRecord(ev_compute, s->compute);
          compute_issued = true;
          progress = true;
        }
      }
    }
    if (finished < static_cast<size_t>(n)) {
      // Nothing to do until the next completion or arrival: back off briefly.
      const double wait = next_arrival < by_arrival.size()
                              ? R[by_arrival[next_arrival]].arrival - (now_s() - host0)
                              : 1.0;
      if (wait > 50e-6) {
        timespec ts{0, 20000};
        nanosleep(&ts, nullptr);
      }
    }
  }
  TSB_CUDA_TRY(cudaStreamSynchronize(st));
  TSB_CUDA_TRY(cudaStreamSynchronize(s->compute));
  cudaEventDestroy(ev_ingest);
  cudaEventDestroy(ev_compute);
  if (status != TSB_OK) return status;

  float last_ms = 0.f;
  for (int64_t i = 0; i < n; ++i) {
    Rt& r = R[i];
    float a = 0.f, b = 0.f, d = 0.f;
    TSB_CUDA_TRY(cudaEventElapsedTime(&a, s->ev_start, r.ev_first));
    TSB_CUDA_TRY(cudaEventElapsedTime(&b, s->ev_start, r.ev_resident));
    TSB_CUDA_TRY(cudaEventElapsedTime(&d, s->ev_start, r.ev_done));
    last_ms = std::max(last_ms, b);
    if (results)
      results[i] = tsb_stage_request{r.id, pick_pos[i], r.deferred, r.n_chunks,
                                     r.n_chunks * chunk_bytes, a, b, d, r.admit_t * 1e3,
                                     r.arrival * 1e3};
  }
  if (stats) {
    stats->bytes = bytes_total;
    stats->device_ms = last_ms;
    stats->wall_ms = (now_s() - wall0) * 1e3;
    stats->ingest_calls = ingest_calls;
    stats->deferred_chunks = deferred_total;
    stats->releases = releases;
    stats->kernel_launches = static_cast<int64_t>(tsb_kernel_launch_count() - launches0);
    stats->verify_mismatches = verify_mismatches;
  }
  return TSB_OK;
}

}  // extern "C"
