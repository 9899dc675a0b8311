// stage.cpp — the real-time load stage (tsb_stage_*).
//
// SimEngine's dispatch rules with real bytes and real time (reference: core/src/engine.cpp):
//   * pick order: the batched GPU scorer (K4/K5) orders the batch by PriorityKey under the chosen
//     policy -- the order best_pending()/admit() would produce for a queue present at one instant
//     (engine.cpp:306-312, 341-355; keys ignore `now`, scheduler.cpp:47);
//   * admission reserves L1 for every planned chunk in block order through the TierLedger-
//     semantics paged allocator (proactive allocation, engine.cpp:419); reservations that do not
//     fit wait FIFO and are granted by later releases (engine.cpp:38-49, 388-397);
//   * a chunk is ingested only once its pages are granted (grant-before-hop, engine.cpp:434-436),
//     requests are served in pick order (pcie_dispatch scans admitted_ in pick order, :427-446);
//   * a request's L1 pages are released when its prefill completes (ComputeDone, :280-282); with
//     prefill disabled, when its last layer is resident;
//   * ControlMode::Coupled (engine.cpp:321-327): one request traverses every stage before the next
//     is admitted.
// The online mode (tsb_stage_run_online) replays arrivals in real time and runs SimEngine's pump
// (try_admit / net_dispatch / pcie_dispatch / try_start_compute to a fixpoint, engine.cpp:290-302)
// against CUDA events instead of a simulated clock.  With an L3 store attached
// (tsb_stage_set_l3) it also runs the network stage for real: blocks start in L3, are granted L2
// slots by a TierLedger(L2) + slot free list at admission (engine.cpp:341-364), are copied
// L3 -> L2 one block at a time by host copy threads (optionally paced to network_bandwidth,
// engine.cpp:405-425), reserve L1 at network dispatch (Proactive, :419) or at NetDone (Reactive,
// :254), and give their L2 slot back when their L2 -> L1 hop completes (:264).  Coupled control
// also holds a request's L2 -> L1 hops until all its network hops are done (:434).
// The simulator's event queue and clock are replaced by CUDA streams and events: ingest on the
// caller's stream, prefill (K6 synthetic, or a caller hook that enqueues a real consumer) on a
// lower-priority compute stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <ctime>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "ledger.h"

using tsb::fail;

namespace {

double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

// Host copy threads for the L3 -> L2 network hop: one block in flight (the reference's single
// network stage, engine.cpp:405-425), split into stripes across the threads.
class NetCopier {
 public:
  explicit NetCopier(int threads) {
    for (int t = 0; t < threads; ++t) workers_.emplace_back([this, t, threads] { loop(t, threads); });
  }
  ~NetCopier() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  void post(const uint8_t* src, uint8_t* dst, size_t bytes) {
    {
      std::lock_guard<std::mutex> g(m_);
      src_ = src;
      dst_ = dst;
      bytes_ = bytes;
      remaining_.store(static_cast<int>(workers_.size()), std::memory_order_release);
      ++gen_;
    }
    cv_.notify_all();
  }
  bool done() const { return remaining_.load(std::memory_order_acquire) == 0; }
  int threads() const { return static_cast<int>(workers_.size()); }

 private:
  void loop(int t, int nt) {
    uint64_t seen = 0;
    for (;;) {
      const uint8_t* src;
      uint8_t* dst;
      size_t bytes;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        src = src_;
        dst = dst_;
        bytes = bytes_;
      }
      const size_t stripe = (bytes / nt + 4095) & ~size_t(4095);
      const size_t lo = std::min(bytes, stripe * t), hi = std::min(bytes, lo + stripe);
      if (hi > lo) std::memcpy(dst + lo, src + lo, hi - lo);
      remaining_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_;
  bool stop_ = false;
  uint64_t gen_ = 0;
  const uint8_t* src_ = nullptr;
  uint8_t* dst_ = nullptr;
  size_t bytes_ = 0;
  std::atomic<int> remaining_{0};
};

// The prefill enqueuer: a host thread of its own.  A real consumer's prefill is thousands of
// kernel launches per batch (cuBLAS + attention per layer); enqueued from the dispatch thread they
// fill the device's launch queue and block that thread, so the link would idle.  Here the stage
// thread only posts "enqueue request i's prefill"; the worker does the waits on the per-layer
// fences, the hook calls and the ComputeDone event, and marks the request enqueued (an event
// queried before it is recorded would read as complete, so completions check the mark first).
class PrefillWorker {
 public:
  PrefillWorker(int device, int64_t n) : device_(device), enqueued_(new std::atomic<uint8_t>[n]) {
    for (int64_t i = 0; i < n; ++i) enqueued_[i].store(0);
    th_ = std::thread([this] { loop(); });
  }
  ~PrefillWorker() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    th_.join();
  }
  void post(int64_t i, std::function<tsb_status()> job) {
    {
      std::lock_guard<std::mutex> g(m_);
      jobs_.emplace_back(i, std::move(job));
    }
    cv_.notify_all();
  }
  bool enqueued(int64_t i) const { return enqueued_[i].load(std::memory_order_acquire) != 0; }
  // Blocks until request i's prefill is enqueued (or the worker failed); returns the status.
  tsb_status wait(int64_t i) {
    std::unique_lock<std::mutex> g(m_);
    done_cv_.wait(g, [&] { return enqueued(i) || status_ != TSB_OK; });
    return status_ != TSB_OK ? fail(status_.load(), msg_) : TSB_OK;
  }
  // Blocks until every posted job ran; returns the first failure.
  tsb_status drain() {
    std::unique_lock<std::mutex> g(m_);
    done_cv_.wait(g, [&] { return (jobs_.empty() && !busy_) || status_ != TSB_OK; });
    return status_ != TSB_OK ? fail(status_.load(), msg_) : TSB_OK;
  }
  tsb_status status() const { return status_; }

 private:
  void loop() {
    cudaSetDevice(device_);
    for (;;) {
      std::pair<int64_t, std::function<tsb_status()>> job;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || !jobs_.empty(); });
        if (jobs_.empty()) return;  // stop requested and nothing left
        job = std::move(jobs_.front());
        jobs_.pop_front();
        busy_ = true;
      }
      const tsb_status prev = status_.load();
      const tsb_status st = prev == TSB_OK ? job.second() : prev;
      {
        std::lock_guard<std::mutex> g(m_);
        busy_ = false;
        if (st != TSB_OK && status_ == TSB_OK) {
          status_ = st;
          msg_ = tsb_last_error();
        }
        if (st == TSB_OK) enqueued_[job.first].store(1, std::memory_order_release);
      }
      done_cv_.notify_all();
    }
  }
  int device_;
  std::unique_ptr<std::atomic<uint8_t>[]> enqueued_;
  std::thread th_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  std::deque<std::pair<int64_t, std::function<tsb_status()>>> jobs_;
  bool stop_ = false, busy_ = false;
  std::atomic<tsb_status> status_{TSB_OK};
  std::string msg_;
};

// Prefill duration of the reference compute stage (engine.cpp:190-212): the measured t_comp for
// replayed requests, else compute_base + per_token * n + quadratic * n^2.
double compute_seconds(const tsb_queue* q, int64_t i, const tsb_cluster* c, int64_t compute_tokens) {
  if (q->flags && (q->flags[i] & TSB_HAS_MEASURED)) return q->measured_t_comp[i];
  const auto ct = static_cast<double>(compute_tokens);
  return c->compute_base + c->compute_per_token * ct + c->compute_quadratic * ct * ct;
}

}  // namespace

struct tsb_stage {
  tsb_l1* l1 = nullptr;
  tsb_pool* pool = nullptr;      // L2 (pinned host) pool
  tsb_pool* hbm_pool = nullptr;  // HBM tier: slots < 0 name slot ~slot of this pool
  tsb_pool* l3 = nullptr;        // online mode: blocks start here; `pool` becomes the L2 slot cache
  NetCopier* net = nullptr;
  tsb_prefill_hook hook = nullptr;
  void* hook_user = nullptr;
  tsb_kv_shape shape{};
  int device = 0;
  tsb_scorer* scorer = nullptr;
  cudaStream_t compute = nullptr;
  bool own_compute = true;  // false: the caller's stream (tsb_stage_set_compute_stream)
  std::vector<cudaEvent_t> timing_pool;  // 3 per request, grown on demand
  std::vector<cudaEvent_t> layer_ev;     // per-layer fences of compute-only requests
  std::vector<cudaEvent_t> layer_pool;   // per-(request, layer) fences, grown on demand
  std::vector<cudaEvent_t> call_pool;    // per ingest call (online PcieDone / trace), grown on demand
  cudaEvent_t ev_start = nullptr;
  std::vector<tsb_trace_row> trace;
  uint64_t seq = 0;
};

namespace {


tsb_status grow_events(std::vector<cudaEvent_t>& v, size_t n, unsigned flags) {
  while (v.size() < n) {
    cudaEvent_t e;
    TSB_CUDA_TRY(cudaEventCreateWithFlags(&e, flags));
    v.push_back(e);
  }
  return TSB_OK;
}

// The ingest mode a run uses: the caller's choice; AUTO resolves per call (CE + K2 for host
// pools).  While a prefill shares the GPU the stage keeps CE + K2: with per-layer fences it holds
// 54.8-55.1 GB/s beside GEMMs and attention, and the real consumer runs 1% faster beside it than
// beside CE-direct's page writes (repo:profiles/r02_stage_mode_ab_strips.jsonl).
int ingest_mode(const tsb_stage*, const tsb_stage_options* opt) { return opt->mode; }

// While a prefill shares the GPU, the stage caps CE staging groups at 128 MiB (unless the caller
// set a cap on the L1): with K6 at 4 us/token, 512 MiB groups delay the prefill start of each
// request (mean TTFT 865 vs 842 ms, DES error 8.5% vs 2.9%) at the same ingest rate and the same
// real-consumer TTFT; 64 MiB groups start to cost link rate (repo:profiles/r02_ce_group_under_prefill.jsonl).
constexpr int64_t kPrefillGroupBytes = 128ll << 20;

class GroupCapScope {
 public:
  GroupCapScope(tsb_l1* l1, bool prefill) : l1_(l1), prev_(tsb_l1_ce_group_bytes(l1)) {
    if (prefill && prev_ == 0) tsb_l1_set_ce_group_bytes(l1_, kPrefillGroupBytes);
  }
  ~GroupCapScope() { tsb_l1_set_ce_group_bytes(l1_, prev_); }

 private:
  tsb_l1* l1_;
  int64_t prev_;
};

// Enqueues a request's prefill on the compute stream: for each layer, wait on its fence (may be
// null = no wait), then the caller's hook or the K6 burner for that layer's share of `secs`.
tsb_status enqueue_prefill(tsb_stage* s, int64_t q_index, int32_t bt_row, double secs,
                           const std::vector<cudaEvent_t>& fences, int ctas) {
  const int64_t L = s->shape.layers;
  const auto per_layer_ns = static_cast<uint64_t>(secs * 1e9 / static_cast<double>(L));
  for (int64_t l = 0; l < L; ++l) {
    if (fences[static_cast<size_t>(l)]) TSB_CUDA_TRY(cudaStreamWaitEvent(s->compute, fences[l], 0));
    if (s->hook) {
      if (s->hook(s->hook_user, q_index, bt_row, l, s->compute) != 0)
        return fail(TSB_VALIDATION, "stage: prefill hook failed at request index " +
                                        std::to_string(q_index) + " layer " + std::to_string(l));
    } else {
      for (uint64_t done = 0; done < per_layer_ns; done += 250000)
        TSB_CUDA_TRY(tsb::launch_prefill_burn(std::min<uint64_t>(250000, per_layer_ns - done), ctas,
                                              nullptr, s->compute));
    }
  }
  return TSB_OK;
}

}  // namespace

extern "C" {

tsb_status tsb_stage_create(tsb_l1* l1, tsb_pool* pool, tsb_stage** out) {
  auto* s = new tsb_stage();
  s->l1 = l1;
  s->pool = pool;
  tsb_status st = tsb_l1_shape(l1, &s->shape);
  if (st != TSB_OK) {
    delete s;
    return st;
  }
  s->device = tsb_l1_device(l1);
  tsb::DeviceGuard dg(s ? s->device : -1);
  int lo = 0, hi = 0;
  cudaError_t e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
  // Prefill gets the LOWEST priority so the ingest scatter kernels interleave ahead of it.
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&s->compute, cudaStreamNonBlocking, lo);
  if (e == cudaSuccess) e = cudaEventCreate(&s->ev_start);
  if (e != cudaSuccess) {
    tsb_stage_destroy(s);
    return tsb::cuda_fail(e, "tsb_stage_create");
  }
  st = grow_events(s->layer_ev, static_cast<size_t>(s->shape.layers), cudaEventDisableTiming);
  if (st == TSB_OK) st = tsb_scorer_create(s->device, 1024, &s->scorer);
  if (st != TSB_OK) {
    tsb_stage_destroy(s);
    return st;
  }
  *out = s;
  return TSB_OK;
}

tsb_status tsb_stage_set_hbm_tier(tsb_stage* s, tsb_pool* hbm_pool) {
  if (hbm_pool && tsb_pool_chunk_bytes(hbm_pool) != tsb_pool_chunk_bytes(s->pool))
    return fail(TSB_VALIDATION, "stage: the HBM tier's chunk geometry differs from the L2 pool's");
  s->hbm_pool = hbm_pool;
  return TSB_OK;
}

tsb_status tsb_stage_set_l3(tsb_stage* s, tsb_pool* l3, int copy_threads) {
  if (l3 && tsb_pool_chunk_bytes(l3) != tsb_pool_chunk_bytes(s->pool))
    return fail(TSB_VALIDATION, "stage: the L3 store's chunk geometry differs from the L2 pool's");
  if (l3 && tsb_pool_location_of(l3) != TSB_POOL_HOST)
    return fail(TSB_VALIDATION, "stage: the L3 store must be host memory");
  if (l3 && tsb_pool_location_of(s->pool) != TSB_POOL_HOST)
    return fail(TSB_VALIDATION, "stage: with an L3 store the L2 pool must be host memory");
  delete s->net;
  s->net = nullptr;
  s->l3 = l3;
  if (l3) s->net = new NetCopier(std::max(1, std::min(copy_threads > 0 ? copy_threads : 4, 32)));
  return TSB_OK;
}

tsb_status tsb_stage_set_prefill_hook(tsb_stage* s, tsb_prefill_hook hook, void* user) {
  s->hook = hook;
  s->hook_user = user;
  return TSB_OK;
}

void* tsb_stage_compute_stream(tsb_stage* s) { return s->compute; }

tsb_status tsb_stage_set_compute_stream(tsb_stage* s, void* stream) {
  tsb::DeviceGuard dg(s ? s->device : -1);
  TSB_CUDA_TRY(cudaStreamSynchronize(s->compute));
  if (s->own_compute) TSB_CUDA_TRY(cudaStreamDestroy(s->compute));
  if (stream) {
    s->compute = static_cast<cudaStream_t>(stream);
    s->own_compute = false;
    return TSB_OK;
  }
  int lo = 0, hi = 0;
  TSB_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  TSB_CUDA_TRY(cudaStreamCreateWithPriority(&s->compute, cudaStreamNonBlocking, lo));
  s->own_compute = true;
  return TSB_OK;
}

void tsb_stage_destroy(tsb_stage* s) {
  if (!s) return;
  tsb::DeviceGuard dg(s ? s->device : -1);
  delete s->net;
  for (auto e : s->timing_pool) cudaEventDestroy(e);
  for (auto e : s->layer_ev) cudaEventDestroy(e);
  for (auto e : s->layer_pool) cudaEventDestroy(e);
  for (auto e : s->call_pool) cudaEventDestroy(e);
  if (s->ev_start) cudaEventDestroy(s->ev_start);
  if (s->compute) {
    cudaStreamSynchronize(s->compute);
    if (s->own_compute) cudaStreamDestroy(s->compute);
  }
  tsb_scorer_destroy(s->scorer);
  delete s;
}

tsb_status tsb_stage_trace(tsb_stage* s, tsb_trace_row* out, int64_t cap, int64_t* n) {
  *n = static_cast<int64_t>(s->trace.size());
  for (int64_t i = 0; i < *n && i < cap; ++i) out[i] = s->trace[i];
  return TSB_OK;
}

}  // extern "C"

namespace {

// Common per-call setup of both modes: plans (types.cpp:85-101), slot checks, capacity checks
// (engine.cpp:213-217), duplicate ids (engine.cpp:126-127).
struct Plan {
  int64_t id = 0, n_chunks = 0, compute_tokens = 0;
  const int64_t* slots = nullptr;
};

tsb_status make_plans(tsb_stage* s, int64_t n, const tsb_queue* q, const tsb_cluster* c,
                      const int64_t* slot_offsets, const int64_t* slots, int64_t chunk_bytes,
                      bool use_l3, std::vector<Plan>* plans,
                      std::unordered_map<int64_t, size_t>* by_id) {
  plans->assign(static_cast<size_t>(n), Plan{});
  const int64_t l1_capacity = tsb_l1_capacity(s->l1);
  const int64_t src_slots = tsb_pool_slots(use_l3 ? s->l3 : s->pool);
  // L2 (L3 mode) is counted in whole pool slots, as the online stage's TierLedger(L2) grants them
  int64_t l2_slots = 0;
  if (use_l3) l2_slots = std::min<int64_t>(c->l2_capacity / tsb_pool_chunk_bytes(s->pool), tsb_pool_slots(s->pool));
  for (int64_t i = 0; i < n; ++i) {
    int64_t cached = 0, compute = 0, nb = 0, bt = 0, bb = 0;
    TSB_TRY(tsb_derive_block_plan(q, i, c, &cached, &compute, &nb, &bt, &bb));
    Plan& r = (*plans)[static_cast<size_t>(i)];
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
      if (use_l3 && sl < 0)
        return fail(TSB_VALIDATION, "stage: with an L3 store every slot names an L3 chunk (no HBM tier)");
      const bool ok = sl >= 0 ? sl < src_slots : (s->hbm_pool && ~sl < tsb_pool_slots(s->hbm_pool));
      if (!ok) return fail(TSB_VALIDATION, "stage: pool slot out of range");
    }
    if (nb * chunk_bytes > l1_capacity || (use_l3 && nb > l2_slots))
      return fail(TSB_CAPACITY, "request " + std::to_string(r.id) + ": " +
                                    std::to_string(nb * chunk_bytes) +
                                    " resident bytes can never fit");
    if (!by_id->emplace(r.id, static_cast<size_t>(i)).second)
      return fail(TSB_VALIDATION, "run_simulation: duplicate request id " + std::to_string(r.id));
  }
  return TSB_OK;
}

}  // namespace

extern "C" {

tsb_status tsb_stage_run(tsb_stage* s, int64_t n, const tsb_queue* q, const tsb_cluster* c,
                         const double models[4], const int64_t* slot_offsets,
                         const int64_t* slots, const tsb_stage_options* opt, void* stream,
                         tsb_stage_request* results, tsb_stage_stats* stats) {
  tsb::DeviceGuard dg(s ? s->device : -1);
  const double wall0 = now_s();
  const uint64_t launches0 = tsb_kernel_launch_count();
  auto st = static_cast<cudaStream_t>(stream);
  const int64_t L = s->shape.layers;
  int64_t chunk_bytes_full = 0, page_bytes = 0, chunk_bytes = 0;
  TSB_TRY(tsb_kv_shape_info(&s->shape, &chunk_bytes_full, &page_bytes, &chunk_bytes));
  TSB_TRY(tsb_cluster_validate(c));
  if (c->block_size_tokens != s->shape.chunk_tokens)
    return fail(TSB_VALIDATION, "stage: cluster block_size_tokens must equal the KV chunk_tokens");
  if (s->l3)
    return fail(TSB_UNSUPPORTED, "stage: the L3 network stage runs in tsb_stage_run_online only");
  const bool coupled = c->control_mode == 0;
  const int mode = ingest_mode(s, opt);
  GroupCapScope group_cap(s->l1, opt->prefill || s->hook);
  s->trace.clear();
  s->seq = 0;
  auto row = [&](double t, int kind, int stg, int tier, int64_t rid, int32_t blk, int64_t bytes) {
    if (opt->record_trace) s->trace.push_back({t, s->seq++, kind, stg, tier, blk, rid, bytes});
  };

  std::vector<Plan> plans;
  std::unordered_map<int64_t, size_t> by_id;
  TSB_TRY(make_plans(s, n, q, c, slot_offsets, slots, chunk_bytes, false, &plans, &by_id));
  struct ReqRt {
    int32_t row = -1;
    std::vector<int32_t> ready;  // granted, not yet ingested (block order)
    int64_t issued = 0;
    int32_t deferred = 0;
    bool finished_issue = false;
    bool read_by_copy = false;  // reuse_l1: ev_reader guards this request's pages until copied
    cudaEvent_t ev_first = nullptr, ev_resident = nullptr, ev_done = nullptr, ev_begin = nullptr;
    cudaEvent_t ev_reader = nullptr;
  };
  std::vector<ReqRt> reqs(static_cast<size_t>(n));
  TSB_TRY(grow_events(s->timing_pool, static_cast<size_t>(5 * n), cudaEventDefault));
  for (int64_t i = 0; i < n; ++i) {
    reqs[i].ev_first = s->timing_pool[5 * i];
    reqs[i].ev_resident = s->timing_pool[5 * i + 1];
    reqs[i].ev_done = s->timing_pool[5 * i + 2];
    reqs[i].ev_begin = s->timing_pool[5 * i + 3];
    reqs[i].ev_reader = s->timing_pool[5 * i + 4];
  }
  // reuse_l1: L2 slot -> a live request's (row, chunk) whose pages hold that chunk (issued).
  struct Holder {
    int64_t req;
    int32_t row, chunk;
  };
  std::unordered_map<int64_t, std::vector<Holder>> holders;  // every live holder, oldest first
  int64_t reused_chunks = 0;

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
  std::vector<cudaEvent_t> call_events;  // trace only: one per ingest call

  const bool with_prefill = opt->prefill || s->hook;
  std::unique_ptr<PrefillWorker> worker;
  if (with_prefill) worker = std::make_unique<PrefillWorker>(s->device, n);

  // Once a request's last chunk is dispatched: ev_first / ev_resident were recorded by that ingest
  // call (or here for an empty plan); now the prefill (posted to the worker) and ev_done.
  auto finish_request_events = [&](int64_t i) -> tsb_status {
    ReqRt& r = reqs[i];
    const Plan& p = plans[i];
    if (p.n_chunks == 0) {
      TSB_CUDA_TRY(cudaEventRecord(r.ev_begin, st));
      TSB_CUDA_TRY(cudaEventRecord(r.ev_first, st));
      TSB_CUDA_TRY(cudaEventRecord(r.ev_resident, st));
      for (int64_t l = 0; l < L; ++l) TSB_CUDA_TRY(cudaEventRecord(s->layer_ev[l], st));
    }
    if (opt->prefill || s->hook) {
      std::vector<cudaEvent_t> fences(static_cast<size_t>(L), nullptr);
      fences[0] = opt->layer_events ? r.ev_first : r.ev_resident;
      if (opt->layer_events) {
        for (int64_t l = 1; l + 1 < L; ++l)
          fences[l] = p.n_chunks ? s->layer_pool[static_cast<size_t>(i * L + l)] : s->layer_ev[l];
        if (L > 1) fences[L - 1] = r.ev_resident;
      }
      const double secs = compute_seconds(q, i, c, p.compute_tokens);
      const int32_t row_i = r.row;
      cudaEvent_t ev_done = r.ev_done;
      worker->post(i, [s, i, row_i, secs, fences, ctas, ev_done]() -> tsb_status {
        TSB_TRY(enqueue_prefill(s, i, row_i, secs, fences, ctas));
        TSB_CUDA_TRY(cudaEventRecord(ev_done, s->compute));
        return TSB_OK;
      });
    } else {
      TSB_CUDA_TRY(cudaEventRecord(r.ev_done, st));
    }
    r.finished_issue = true;
    return TSB_OK;
  };

  // pcie_dispatch (engine.cpp:427-446): serve granted chunks of admitted requests in pick order.
  if (opt->layer_events) TSB_TRY(grow_events(s->layer_pool, static_cast<size_t>(n * L), cudaEventDisableTiming));
  auto dispatch = [&]() -> tsb_status {
    bool synced = false;
    for (int64_t k = 0; k < n; ++k) {
      const int64_t i = order[k];
      ReqRt& r = reqs[i];
      const Plan& p = plans[i];
      if (r.finished_issue || r.ready.empty()) continue;
      if (!synced) {
        TSB_TRY(tsb_l1_sync_block_table(s->l1, stream));
        synced = true;
      }
      std::vector<tsb_ingest_item> items;
      std::vector<tsb_page_copy> copies;
      std::vector<int64_t> copy_from;  // holder request of each copy
      items.reserve(r.ready.size());
      for (int32_t ch : r.ready) {
        const int64_t sl = p.slots[ch];
        const auto h = opt->reuse_l1 && sl >= 0 ? holders.find(sl) : holders.end();
        if (h != holders.end() && !h->second.empty()) {
          const Holder& src = h->second.front();
          copies.push_back(tsb_page_copy{src.row, src.chunk, r.row, ch});
          copy_from.push_back(src.req);
        } else {
          items.push_back(tsb_ingest_item{sl, r.row, ch});
        }
        row(now_s() - host0, 4, 1, -1, p.id, ch, chunk_bytes);  // DispatchWake(Pcie)
      }
      if (r.issued == 0) TSB_CUDA_TRY(cudaEventRecord(r.ev_begin, st));  // the request's first hop
      r.issued += static_cast<int64_t>(r.ready.size());
      if (opt->reuse_l1)
        for (int32_t ch : r.ready)
          if (p.slots[ch] >= 0) holders[p.slots[ch]].push_back(Holder{i, r.row, ch});
      r.ready.clear();
      const bool last = r.issued == p.n_chunks;
      if (!copies.empty()) {
        // K8 first: its sources were written by earlier work on this stream; then the link part.
        for (int64_t c0 = 0; c0 < static_cast<int64_t>(copies.size()); c0 += 65536)
          TSB_TRY(tsb_l1_copy_chunks(s->l1, copies.data() + c0,
                                     std::min<int64_t>(65536, static_cast<int64_t>(copies.size()) - c0), 0, L,
                                     stream));
        for (const int64_t h : copy_from) {  // the holders' pages stay until these copies ran
          TSB_CUDA_TRY(cudaEventRecord(reqs[h].ev_reader, st));
          reqs[h].read_by_copy = true;
        }
        reused_chunks += static_cast<int64_t>(copies.size());
        bytes_total += static_cast<int64_t>(copies.size()) * chunk_bytes;  // delivered into L1 all the same
      }
      std::vector<void*> evs;
      void* const* evp = nullptr;
      if (last) {
        // Timing events double as the layer-0 and last-layer fences; the layers between get this
        // request's own fences (its prefill is enqueued after later requests' ingest).
        evs.assign(static_cast<size_t>(L), nullptr);
        if (opt->layer_events)
          for (int64_t l = 1; l + 1 < L; ++l) evs[l] = s->layer_pool[static_cast<size_t>(i * L + l)];
        evs[0] = r.ev_first;
        evs[L - 1] = r.ev_resident;
        evp = evs.data();
      }
      TSB_TRY(tsb_ingest_tiered(s->l1, s->pool, s->hbm_pool, items.data(),
                                static_cast<int64_t>(items.size()), 0, L, mode, stream, evp));
      if (last && (L == 1 || !copies.empty())) TSB_CUDA_TRY(cudaEventRecord(r.ev_first, st));
      if (last && !copies.empty()) {  // the fences must also cover the replicated chunks
        for (int64_t l = 1; opt->layer_events && l + 1 < L; ++l)
          TSB_CUDA_TRY(cudaEventRecord(s->layer_pool[static_cast<size_t>(i * L + l)], st));
        TSB_CUDA_TRY(cudaEventRecord(r.ev_resident, st));
      }
      if (opt->record_trace) {
        if (call_events.size() >= 4096) return fail(TSB_CAPACITY, "stage: more than 4096 traced ingest calls");
        TSB_TRY(grow_events(s->call_pool, call_events.size() + 1, cudaEventDefault));
        cudaEvent_t ce = s->call_pool[call_events.size()];
        TSB_CUDA_TRY(cudaEventRecord(ce, st));
        call_events.push_back(ce);
        for (const auto& it : items)  // TransferDone(Pcie); time filled in after the run
          row(-static_cast<double>(call_events.size()), 1, 1, -1, p.id, it.chunk_index, chunk_bytes);
      }
      ++ingest_calls;
      bytes_total += static_cast<int64_t>(items.size()) * chunk_bytes;
      // Completion right away: without prefill ev_done is recorded now; with prefill the request
      // is posted to the enqueue thread, so this loop never waits on the consumer.
      if (last) TSB_TRY(finish_request_events(i));
    }
    return TSB_OK;
  };

  // admit (engine.cpp:341-355): reserve L1 for every planned chunk of a request.
  auto admit = [&](int64_t i) -> tsb_status {
    ReqRt& r = reqs[i];
    const Plan& p = plans[i];
    for (int64_t ch = 0; ch < p.n_chunks; ++ch) {
      int granted = 0;
      TSB_TRY(tsb_l1_request(s->l1, p.id, static_cast<int32_t>(ch), chunk_bytes, &granted, &r.row));
      if (granted) {
        r.ready.push_back(static_cast<int32_t>(ch));
        row(now_s() - host0, 2, -1, 2, p.id, static_cast<int32_t>(ch), chunk_bytes);
      } else {
        ++r.deferred;
        ++deferred_total;
      }
    }
    if (p.n_chunks == 0) TSB_TRY(finish_request_events(i));
    return TSB_OK;
  };

  // ComputeDone (engine.cpp:274-283): wait, optionally verify, release L1 (FIFO grants), and
  // dispatch what the grants made ready.
  auto complete = [&](int64_t i) -> tsb_status {
    ReqRt& r = reqs[i];
    const Plan& p = plans[i];
    if (worker) TSB_TRY(worker->wait(i));  // its ComputeDone event is recorded
    TSB_CUDA_TRY(cudaEventSynchronize(r.ev_done));
    if (opt->verify_seed && p.n_chunks > 0) {
      std::vector<tsb_ingest_item> items;
      // both tiers hold the synthetic pattern of the seed at their own slot index
      for (int64_t ch = 0; ch < p.n_chunks; ++ch)
        items.push_back(tsb_ingest_item{p.slots[ch] < 0 ? ~p.slots[ch] : p.slots[ch], r.row,
                                        static_cast<int32_t>(ch)});
      uint64_t mm = 0;
      TSB_TRY(tsb_l1_verify_synthetic(s->l1, items.data(), p.n_chunks, 0, L, opt->verify_seed,
                                      tsb_pool_chunk_bytes(s->pool), stream, &mm));
      verify_mismatches += mm;
    }
    row(now_s() - host0, 3, 2, -1, p.id, -1, p.compute_tokens * c->bytes_per_token);
    if (opt->reuse_l1) {  // its pages stop being a copy source; pending copies from them finish first
      for (int64_t ch = 0; ch < p.n_chunks; ++ch) {
        const auto h = p.slots[ch] >= 0 ? holders.find(p.slots[ch]) : holders.end();
        if (h == holders.end()) continue;
        auto& v = h->second;
        v.erase(std::remove_if(v.begin(), v.end(), [&](const Holder& x) { return x.req == i; }), v.end());
      }
      if (r.read_by_copy) TSB_CUDA_TRY(cudaEventSynchronize(r.ev_reader));
    }
    if (r.row >= 0) {
      std::vector<tsb_grant> grants(static_cast<size_t>(tsb_l1_deferred(s->l1)) + 1);
      int64_t ng = 0;
      TSB_TRY(tsb_l1_release_request(s->l1, p.id, grants.data(), static_cast<int64_t>(grants.size()), &ng));
      ++releases;
      const double t = now_s() - host0;
      for (int64_t g = 0; g < ng; ++g) {
        ReqRt& w = reqs[by_id.at(grants[g].request_id)];
        w.ready.push_back(grants[g].block_index);
        row(t, 2, -1, 2, grants[g].request_id, grants[g].block_index, grants[g].bytes);
      }
      TSB_TRY(dispatch());
    }
    return TSB_OK;
  };

  tsb_status status = TSB_OK;
  if (coupled) {
    // ControlMode::Coupled (engine.cpp:321-327): admit the next request only when the previous
    // one has traversed every stage (its prefill is done and its pages are released).
    for (int64_t k = 0; k < n && status == TSB_OK; ++k) {
      status = admit(order[k]);
      if (status == TSB_OK) status = dispatch();
      if (status == TSB_OK) status = complete(order[k]);
    }
  } else {
    // Decoupled: admit everything in pick order up front; then complete requests in pick order,
    // each release granting deferred reservations whose chunks are dispatched right away so the
    // link never idles while the host waits.
    for (int64_t k = 0; k < n && status == TSB_OK; ++k) status = admit(order[k]);
    if (status == TSB_OK) status = dispatch();
    for (int64_t k = 0; k < n && status == TSB_OK; ++k) {
      if (!reqs[order[k]].finished_issue) {
        status = fail(TSB_CAPACITY, "stage: request " + std::to_string(plans[order[k]].id) +
                                        " is blocked on L1 pages held by later requests");
        break;
      }
      status = complete(order[k]);
    }
  }
  if (worker && status == TSB_OK) status = worker->drain();
  worker.reset();  // joins: no hook runs after this call returns
  if (status != TSB_OK) {
    // Leave nothing in flight and no reservation held: drain both streams, then release every
    // request's L1 pages (the allocator returns to its pre-call state).
    const std::string msg = tsb_last_error();
    cudaStreamSynchronize(st);
    cudaStreamSynchronize(s->compute);
    for (int64_t i = 0; i < n; ++i) {
      if (reqs[i].row < 0 && reqs[i].deferred == 0) continue;
      std::vector<tsb_grant> grants(static_cast<size_t>(tsb_l1_deferred(s->l1)) + 1);
      int64_t ng = 0;
      tsb_l1_release_request(s->l1, plans[i].id, grants.data(), static_cast<int64_t>(grants.size()), &ng);
    }
    return fail(status, msg);
  }
  TSB_CUDA_TRY(cudaStreamSynchronize(st));

  // ---- results --------------------------------------------------------------------------------
  float last_ms = 0.f;
  for (int64_t i = 0; i < n; ++i) {
    ReqRt& r = reqs[i];
    float a = 0.f, b = 0.f, d = 0.f, g = 0.f;
    TSB_CUDA_TRY(cudaEventElapsedTime(&a, s->ev_start, r.ev_first));
    TSB_CUDA_TRY(cudaEventElapsedTime(&b, s->ev_start, r.ev_resident));
    TSB_CUDA_TRY(cudaEventElapsedTime(&d, s->ev_start, r.ev_done));
    TSB_CUDA_TRY(cudaEventElapsedTime(&g, s->ev_start, r.ev_begin));
    last_ms = std::max(last_ms, b);
    if (results)
      results[i] = tsb_stage_request{plans[i].id, static_cast<int32_t>(pos_of[i]), r.deferred,
                                     plans[i].n_chunks, plans[i].n_chunks * chunk_bytes, a, b, d, 0.0, 0.0,
                                     g, plans[i].n_chunks * s->shape.chunk_tokens, plans[i].compute_tokens};
  }
  if (opt->record_trace) {
    for (auto& tr : s->trace) {
      if (tr.time < 0) {
        float ms = 0.f;
        TSB_CUDA_TRY(cudaEventElapsedTime(&ms, s->ev_start, call_events[static_cast<size_t>(-tr.time) - 1]));
        tr.time = ms * 1e-3;
      }
    }
  }
  if (stats) {
    *stats = tsb_stage_stats{};
    stats->bytes = bytes_total;
    stats->device_ms = last_ms;
    stats->wall_ms = (now_s() - wall0) * 1e3;
    stats->ingest_calls = ingest_calls;
    stats->deferred_chunks = deferred_total;
    stats->releases = releases;
    stats->kernel_launches = static_cast<int64_t>(tsb_kernel_launch_count() - launches0);
    stats->verify_mismatches = verify_mismatches;
    stats->reused_chunks = reused_chunks;
  }
  return TSB_OK;
}

// ------------------------------------------------------------------------------------------------
// Online mode: SimEngine's event loop (engine.cpp:140-158, 290-302) in real time.
// ------------------------------------------------------------------------------------------------
tsb_status tsb_stage_run_online(tsb_stage* s, int64_t n, const tsb_queue* q,
                                const tsb_cluster* c, const double models[4],
                                const int64_t* slot_offsets, const int64_t* slots,
                                const tsb_stage_options* opt, void* stream,
                                tsb_stage_request* results, tsb_stage_stats* stats) {
  tsb::DeviceGuard dg(s ? s->device : -1);
  const double wall0 = now_s();
  const uint64_t launches0 = tsb_kernel_launch_count();
  auto st = static_cast<cudaStream_t>(stream);
  const int64_t L = s->shape.layers;
  int64_t chunk_bytes_full = 0, page_bytes = 0, chunk_bytes = 0;
  TSB_TRY(tsb_kv_shape_info(&s->shape, &chunk_bytes_full, &page_bytes, &chunk_bytes));
  TSB_TRY(tsb_cluster_validate(c));
  if (c->block_size_tokens != s->shape.chunk_tokens)
    return fail(TSB_VALIDATION, "stage: cluster block_size_tokens must equal the KV chunk_tokens");
  const bool use_l3 = s->l3 != nullptr;
  const bool coupled = c->control_mode == 0;
  const bool reactive = c->allocation_mode == 1;
  const bool reuse = opt->reuse_l1 != 0;
  if (reuse && use_l3)
    return fail(TSB_UNSUPPORTED, "stage: reuse_l1 with an L3 store (blocks pass through L2 slots, not pool slots)");
  const int mode = ingest_mode(s, opt);
  GroupCapScope group_cap(s->l1, opt->prefill || s->hook);
  const int64_t l2_slot_bytes = tsb_pool_chunk_bytes(s->pool);
  s->trace.clear();
  s->seq = 0;
  if (n == 0) {
    if (stats) *stats = tsb_stage_stats{};
    return TSB_OK;
  }
  std::vector<Plan> plans;
  std::unordered_map<int64_t, size_t> by_id;
  TSB_TRY(make_plans(s, n, q, c, slot_offsets, slots, chunk_bytes, use_l3, &plans, &by_id));

  struct Blk {
    int64_t l2_slot = -1;  // L3 mode: the L2 slot this block was granted
    bool l2_granted = false, l1_granted = false, net_done = false, pcie_issued = false;
  };
  struct Rt {
    std::vector<Blk> blk;
    int32_t row = -1, deferred = 0;
    int64_t next_net = 0, next_pcie = 0, net_done = 0, pcie_issued = 0, pcie_done = 0;
    bool arrived = false, admitted = false, compute_ready = false, started = false, finished = false;
    bool released = false;      // its L1 pages went back to the allocator
    bool read_by_copy = false;  // reuse_l1: ev_reader guards its pages until K8 has read them
    double arrival = 0.0, admit_t = 0.0;
    cudaEvent_t ev_first = nullptr, ev_resident = nullptr, ev_done = nullptr, ev_begin = nullptr;
    cudaEvent_t ev_reader = nullptr;
  };
  std::vector<Rt> R(static_cast<size_t>(n));
  double first_arrival = q->arrival[0];
  for (int64_t i = 0; i < n; ++i) first_arrival = std::min(first_arrival, q->arrival[i]);
  TSB_TRY(grow_events(s->timing_pool, static_cast<size_t>(5 * n), cudaEventDefault));
  for (int64_t i = 0; i < n; ++i) {
    Rt& r = R[i];
    r.blk.resize(static_cast<size_t>(plans[i].n_chunks));
    r.arrival = q->arrival[i] - first_arrival;
    r.ev_first = s->timing_pool[5 * i];
    r.ev_resident = s->timing_pool[5 * i + 1];
    r.ev_done = s->timing_pool[5 * i + 2];
    r.ev_begin = s->timing_pool[5 * i + 3];
    r.ev_reader = s->timing_pool[5 * i + 4];
  }
  // reuse_l1: pool slot -> live requests whose pages hold that chunk (hop issued), oldest first.
  struct Holder {
    size_t req;
    int32_t row, chunk;
  };
  std::unordered_map<int64_t, std::vector<Holder>> holders;
  std::vector<size_t> release_wait;  // ComputeDone seen, pages still being read by K8 copies
  int64_t reused_chunks = 0;
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

  // L2 tier (L3 mode): TierLedger(L2) over the pool's slots + a FIFO slot free list.
  tsb::Ledger l2(1, use_l3 ? std::min<int64_t>(c->l2_capacity / l2_slot_bytes, tsb_pool_slots(s->pool)) * l2_slot_bytes
                           : 1);
  std::deque<int64_t> l2_free;
  if (use_l3)
    for (int64_t k = 0; k < tsb_pool_slots(s->pool); ++k) l2_free.push_back(k);

  struct Call {  // one L2 -> L1 ingest call: its blocks complete together (PcieDone)
    cudaEvent_t ev;
    size_t req;
    std::vector<int32_t> blocks;
  };
  std::deque<Call> calls;
  size_t call_slot = 0;
  const int ctas = opt->prefill_ctas > 0 ? opt->prefill_ctas : 148;
  int64_t ingest_calls = 0, deferred_total = 0, releases = 0, bytes_total = 0, net_blocks = 0, l2_deferred = 0;
  uint64_t verify_mismatches = 0;
  std::vector<size_t> pending, admitted;
  size_t admitted_head = 0, next_arrival = 0, finished = 0;
  int64_t pick = 0, unissued_net = 0, active = 0;
  std::vector<int32_t> pick_pos(static_cast<size_t>(n), -1);
  bool net_busy = false, compute_busy = false;
  size_t net_req = 0;
  int64_t net_blk = 0;
  double net_ready_at = 0.0;

  PrefillWorker worker(s->device, n);  // the compute stage's enqueuer (see PrefillWorker)
  TSB_CUDA_TRY(cudaEventRecord(s->ev_start, st));
  const double host0 = now_s();
  auto now = [&] { return now_s() - host0; };
  auto row = [&](int kind, int stg, int tier, int64_t rid, int32_t blk, int64_t bytes) {
    if (opt->record_trace) s->trace.push_back({now(), s->seq++, kind, stg, tier, blk, rid, bytes});
  };
  auto done = [](cudaEvent_t e) { return cudaEventQuery(e) == cudaSuccess; };
  std::vector<tsb_grant> grants(64);
  double last_progress = now();

  auto grant_l1 = [&](size_t i, int32_t b) {
    R[i].blk[static_cast<size_t>(b)].l1_granted = true;
    row(2, -1, 2, plans[i].id, b, chunk_bytes);
  };
  auto request_l1 = [&](size_t i, int32_t b) -> tsb_status {
    int granted = 0;
    TSB_TRY(tsb_l1_request(s->l1, plans[i].id, b, chunk_bytes, &granted, &R[i].row));
    if (granted) {
      grant_l1(i, b);
    } else {
      ++R[i].deferred;
      ++deferred_total;
    }
    return TSB_OK;
  };
  auto grant_l2 = [&](size_t i, int32_t b) {
    Blk& k = R[i].blk[static_cast<size_t>(b)];
    k.l2_granted = true;
    k.l2_slot = l2_free.front();
    l2_free.pop_front();
    row(2, -1, 1, plans[i].id, b, chunk_bytes);
  };
  auto release_l2 = [&](int64_t slot) -> tsb_status {
    l2_free.push_back(slot);
    std::string msg;
    const tsb_status rs = l2.release(l2_slot_bytes, [&](const tsb::Ledger::Pending& p) {
      grant_l2(by_id.at(p.request_id), p.block_index);
    }, &msg);
    return rs == TSB_OK ? TSB_OK : fail(rs, msg);
  };
  // L1 release at ComputeDone (engine.cpp:280-282): FIFO grants to deferred reservations.
  auto release_l1 = [&](size_t i) -> tsb_status {
    Rt& r = R[i];
    r.released = true;
    if (r.row < 0 && r.deferred == 0) return TSB_OK;
    int64_t ng = 0;
    grants.resize(static_cast<size_t>(tsb_l1_deferred(s->l1)) + 1);
    TSB_TRY(tsb_l1_release_request(s->l1, plans[i].id, grants.data(), static_cast<int64_t>(grants.size()), &ng));
    ++releases;
    for (int64_t g = 0; g < ng; ++g) grant_l1(by_id.at(grants[g].request_id), grants[g].block_index);
    return TSB_OK;
  };

  tsb_status status = TSB_OK;
  while (finished < static_cast<size_t>(n) && status == TSB_OK) {
    bool progress = false;
    // ---- handle(): every event that has happened by now (engine.cpp:227-288) ------------------
    while (next_arrival < by_arrival.size() && R[by_arrival[next_arrival]].arrival <= now()) {
      const size_t i = by_arrival[next_arrival++];
      R[i].arrived = true;
      pending.push_back(i);
      row(0, -1, -1, plans[i].id, -1, 0);
      progress = true;
    }
    if (net_busy && s->net->done() && now() >= net_ready_at) {  // NetDone (engine.cpp:242-256)
      Rt& r = R[net_req];
      r.blk[static_cast<size_t>(net_blk)].net_done = true;
      ++r.net_done;
      row(1, 0, -1, plans[net_req].id, static_cast<int32_t>(net_blk), chunk_bytes);
      if (reactive && (status = request_l1(net_req, static_cast<int32_t>(net_blk))) != TSB_OK) break;
      net_busy = false;
      progress = true;
    }
    while (!calls.empty() && done(calls.front().ev)) {  // PcieDone (engine.cpp:258-272)
      Call cl = std::move(calls.front());
      calls.pop_front();
      Rt& r = R[cl.req];
      for (int32_t b : cl.blocks) {
        row(1, 1, -1, plans[cl.req].id, b, chunk_bytes);
        ++r.pcie_done;
        if (use_l3 && (status = release_l2(r.blk[static_cast<size_t>(b)].l2_slot)) != TSB_OK) break;
      }
      if (status != TSB_OK) break;
      if (r.pcie_done == plans[cl.req].n_chunks) r.compute_ready = true;
      progress = true;
    }
    if (status != TSB_OK) break;
    if ((status = worker.status()) != TSB_OK) {
      status = worker.drain();
      break;
    }
    for (size_t k = admitted_head; k < admitted.size(); ++k) {  // ComputeDone (engine.cpp:274-283)
      const size_t i = admitted[k];
      Rt& r = R[i];
      if (!r.started || r.finished || !worker.enqueued(static_cast<int64_t>(i)) || !done(r.ev_done)) continue;
      r.finished = true;
      ++finished;
      --active;
      compute_busy = false;
      progress = true;
      row(3, 2, -1, plans[i].id, -1, plans[i].compute_tokens * c->bytes_per_token);
      if (opt->verify_seed && plans[i].n_chunks > 0) {  // opt-in check (synchronises the stream)
        std::vector<tsb_ingest_item> items;
        for (int64_t ch = 0; ch < plans[i].n_chunks; ++ch) {
          const int64_t sl = plans[i].slots[ch];
          items.push_back(tsb_ingest_item{sl < 0 ? ~sl : sl, r.row, static_cast<int32_t>(ch)});
        }
        uint64_t mm = 0;
        if ((status = tsb_l1_verify_synthetic(s->l1, items.data(), plans[i].n_chunks, 0, L, opt->verify_seed,
                                              tsb_pool_chunk_bytes(s->pool), stream, &mm)) != TSB_OK)
          break;
        verify_mismatches += mm;
      }
      if (reuse) {  // its pages stop being a copy source; copies already issued from them finish first
        for (int64_t ch = 0; ch < plans[i].n_chunks; ++ch) {
          const auto h = plans[i].slots[ch] >= 0 ? holders.find(plans[i].slots[ch]) : holders.end();
          if (h == holders.end()) continue;
          auto& v = h->second;
          v.erase(std::remove_if(v.begin(), v.end(), [&](const Holder& x) { return x.req == i; }), v.end());
        }
        if (r.read_by_copy && !done(r.ev_reader)) {
          release_wait.push_back(i);
          continue;
        }
      }
      if ((status = release_l1(i)) != TSB_OK) break;
    }
    if (status != TSB_OK) break;
    for (size_t k = 0; k < release_wait.size() && status == TSB_OK;) {  // deferred ComputeDone releases
      const size_t i = release_wait[k];
      if (!done(R[i].ev_reader)) {
        ++k;
        continue;
      }
      release_wait.erase(release_wait.begin() + static_cast<std::ptrdiff_t>(k));
      status = release_l1(i);
      progress = true;
    }
    if (status != TSB_OK) break;
    while (admitted_head < admitted.size() && R[admitted[admitted_head]].finished) ++admitted_head;

    // ---- pump(): try_admit / net_dispatch / pcie_dispatch / try_start_compute to a fixpoint ---
    bool moved = true;
    while (moved && status == TSB_OK) {
      moved = false;
      // try_admit (engine.cpp:318-339)
      if (!pending.empty()) {
        size_t bi = 0;
        for (size_t k = 1; k < pending.size(); ++k)
          if (key_less(pending[k], pending[bi])) bi = k;
        const size_t i = pending[bi];
        Rt& r = R[i];
        bool can = false;
        if (coupled) {
          can = active == 0;
        } else if (plans[i].n_chunks > 0) {
          if (use_l3) {
            can = !net_busy && unissued_net == 0;
          } else {
            bool backlog = false;  // the first stage is the L2 -> L1 hop: idle with no backlog
            for (size_t k = admitted_head; k < admitted.size(); ++k) {
              const Rt& a = R[admitted[k]];
              if (a.admitted && a.pcie_issued < static_cast<int64_t>(a.blk.size())) backlog = true;
            }
            can = !backlog && calls.empty();
          }
        } else {
          bool ready_waiting = false;
          for (size_t k = admitted_head; k < admitted.size(); ++k)
            if (R[admitted[k]].compute_ready && !R[admitted[k]].started) ready_waiting = true;
          can = !compute_busy && !ready_waiting;
        }
        if (can) {  // admit (engine.cpp:341-355)
          pending.erase(pending.begin() + static_cast<std::ptrdiff_t>(bi));
          r.admitted = true;
          r.admit_t = now();
          pick_pos[i] = static_cast<int32_t>(pick++);
          admitted.push_back(i);
          ++active;
          const int64_t nb = plans[i].n_chunks;
          if (use_l3) {
            unissued_net += nb;
            for (int64_t b = 0; b < nb; ++b) {  // request_l2 (engine.cpp:357-362)
              bool granted = false;
              std::string msg;
              const tsb_status rs = l2.request(plans[i].id, static_cast<int32_t>(b), l2_slot_bytes, &granted, &msg);
              if (rs != TSB_OK) {
                status = fail(rs, msg);
                break;
              }
              if (granted) grant_l2(i, static_cast<int32_t>(b));
              else ++l2_deferred;
            }
          } else {
            // Blocks are L2-resident already: the network hop is instantaneous, so proactive and
            // reactive L1 reservation both happen now.
            for (int64_t b = 0; b < nb && status == TSB_OK; ++b) {
              r.blk[static_cast<size_t>(b)].l2_granted = r.blk[static_cast<size_t>(b)].net_done = true;
              status = request_l1(i, static_cast<int32_t>(b));
            }
            r.net_done = nb;
          }
          if (nb == 0) {  // compute-only: ready at admission (engine.cpp:351-354)
            r.compute_ready = true;
            cudaError_t e = cudaEventRecord(r.ev_begin, s->compute);
            if (e == cudaSuccess) e = cudaEventRecord(r.ev_first, s->compute);
            if (e == cudaSuccess) e = cudaEventRecord(r.ev_resident, s->compute);
            if (e != cudaSuccess) status = tsb::cuda_fail(e, "stage: compute-only request events");
          }
          moved = true;
        }
      }
      if (status != TSB_OK) break;
      // net_dispatch (engine.cpp:405-425): one block in flight, first granted block in pick order
      if (use_l3 && !net_busy) {
        for (size_t k = admitted_head; k < admitted.size(); ++k) {
          const size_t i = admitted[k];
          Rt& r = R[i];
          if (r.next_net >= static_cast<int64_t>(r.blk.size())) continue;
          Blk& b = r.blk[static_cast<size_t>(r.next_net)];
          if (!b.l2_granted) continue;
          const int64_t bi = r.next_net++;
          --unissued_net;
          row(4, 0, -1, plans[i].id, static_cast<int32_t>(bi), chunk_bytes);
          if (!reactive && (status = request_l1(i, static_cast<int32_t>(bi))) != TSB_OK) break;
          net_busy = true;
          net_req = i;
          net_blk = bi;
          const double pace = opt->pace_network
                                  ? c->transfer_base_latency + static_cast<double>(l2_slot_bytes) / c->network_bandwidth
                                  : 0.0;
          net_ready_at = now() + pace;
          s->net->post(static_cast<const uint8_t*>(tsb_pool_slot_ptr(s->l3, plans[i].slots[bi])),
                       static_cast<uint8_t*>(tsb_pool_slot_ptr(s->pool, b.l2_slot)),
                       static_cast<size_t>(l2_slot_bytes));
          ++net_blocks;
          moved = true;
          break;
        }
        if (status != TSB_OK) break;
      }
      // pcie_dispatch (engine.cpp:427-446): per admitted request in pick order, its next blocks
      // in block order that are L2-resident and hold L1 pages; one ingest call per request.
      for (size_t k = admitted_head; k < admitted.size() && status == TSB_OK; ++k) {
        const size_t i = admitted[k];
        Rt& r = R[i];
        const int64_t nb = static_cast<int64_t>(r.blk.size());
        if (r.next_pcie >= nb) continue;
        if (coupled && r.net_done < nb) continue;
        std::vector<tsb_ingest_item> items;
        std::vector<tsb_page_copy> copies;
        std::vector<size_t> copy_from;  // holder request of each copy
        std::vector<int32_t> bl;
        while (r.next_pcie < nb) {
          Blk& b = r.blk[static_cast<size_t>(r.next_pcie)];
          if (!b.net_done || !b.l1_granted) break;
          b.pcie_issued = true;
          const int32_t ch = static_cast<int32_t>(r.next_pcie);
          const int64_t src = use_l3 ? b.l2_slot : plans[i].slots[r.next_pcie];
          const auto h = reuse && src >= 0 ? holders.find(src) : holders.end();
          if (h != holders.end() && !h->second.empty()) {
            const Holder& from = h->second.front();
            copies.push_back(tsb_page_copy{from.row, from.chunk, r.row, ch});
            copy_from.push_back(from.req);
          } else {
            items.push_back(tsb_ingest_item{src, r.row, ch});
          }
          bl.push_back(ch);
          row(4, 1, -1, plans[i].id, ch, chunk_bytes);
          ++r.next_pcie;
        }
        if (bl.empty()) continue;
        if ((status = tsb_l1_sync_block_table(s->l1, stream)) != TSB_OK) break;
        if (r.pcie_issued == 0) {
          const cudaError_t e = cudaEventRecord(r.ev_begin, st);
          if (e != cudaSuccess) {
            status = tsb::cuda_fail(e, "stage: ingest begin event");
            break;
          }
        }
        r.pcie_issued += static_cast<int64_t>(bl.size());
        const bool last = r.pcie_issued == nb;
        if (reuse) {
          for (int32_t ch : bl)
            if (plans[i].slots[ch] >= 0) holders[plans[i].slots[ch]].push_back(Holder{i, r.row, ch});
          // K8 first: its sources were written by ingest calls issued earlier on this stream
          for (int64_t c0 = 0; c0 < static_cast<int64_t>(copies.size()) && status == TSB_OK; c0 += 65536)
            status = tsb_l1_copy_chunks(s->l1, copies.data() + c0,
                                        std::min<int64_t>(65536, static_cast<int64_t>(copies.size()) - c0), 0, L,
                                        stream);
          if (status != TSB_OK) break;
          cudaError_t e = cudaSuccess;
          for (const size_t h : copy_from) {  // the holders' pages stay until these copies ran
            if (e == cudaSuccess) e = cudaEventRecord(R[h].ev_reader, st);
            R[h].read_by_copy = true;
          }
          if (e != cudaSuccess) {
            status = tsb::cuda_fail(e, "stage: reuse reader events");
            break;
          }
          reused_chunks += static_cast<int64_t>(copies.size());
          bytes_total += static_cast<int64_t>(copies.size()) * chunk_bytes;  // delivered into L1 all the same
        }
        std::vector<void*> evs;
        if (last) {
          evs.assign(static_cast<size_t>(L), nullptr);
          evs[0] = r.ev_first;
          evs[L - 1] = r.ev_resident;
        }
        if ((status = tsb_ingest_tiered(s->l1, s->pool, s->hbm_pool, items.data(),
                                        static_cast<int64_t>(items.size()), 0, L, mode, stream,
                                        last ? evs.data() : nullptr)) != TSB_OK)
          break;
        if (calls.size() >= 4096) {  // bound the in-flight call list (event slots are reused)
          status = fail(TSB_CAPACITY, "stage: more than 4096 ingest calls in flight");
          break;
        }
        if ((status = grow_events(s->call_pool, std::min<size_t>(call_slot + 1, 4096), cudaEventDefault)) != TSB_OK)
          break;
        cudaEvent_t ce = s->call_pool[call_slot++ % 4096];
        cudaError_t e = cudaSuccess;
        if (last && (L == 1 || !copies.empty())) e = cudaEventRecord(r.ev_first, st);
        if (e == cudaSuccess && last && !copies.empty()) e = cudaEventRecord(r.ev_resident, st);  // covers K8 too
        if (e == cudaSuccess) e = cudaEventRecord(ce, st);
        if (e != cudaSuccess) {
          status = tsb::cuda_fail(e, "stage: ingest call events");
          break;
        }
        calls.push_back(Call{ce, i, std::move(bl)});
        ++ingest_calls;
        bytes_total += static_cast<int64_t>(items.size()) * chunk_bytes;
        moved = true;
      }
      if (status != TSB_OK) break;
      // try_start_compute (engine.cpp:448-473): best key among resident, not started.
      if (!compute_busy) {
        size_t best = SIZE_MAX;
        for (size_t k = admitted_head; k < admitted.size(); ++k) {
          const size_t i = admitted[k];
          if (!R[i].compute_ready || R[i].started) continue;
          if (best == SIZE_MAX || key_less(i, best)) best = i;
        }
        if (best != SIZE_MAX) {
          Rt& r = R[best];
          r.started = true;
          compute_busy = true;
          row(4, 2, -1, plans[best].id, -1, 0);
          std::vector<cudaEvent_t> fences(static_cast<size_t>(L), nullptr);
          fences[0] = r.ev_resident;
          const double secs = opt->prefill || s->hook ? compute_seconds(q, best, c, plans[best].compute_tokens) : 0.0;
          const int64_t bi = static_cast<int64_t>(best);
          const int32_t row_i = r.row;
          cudaEvent_t ev_done = r.ev_done;
          worker.post(bi, [s, bi, row_i, secs, fences, ctas, ev_done]() -> tsb_status {
            TSB_TRY(enqueue_prefill(s, bi, row_i, secs, fences, ctas));
            TSB_CUDA_TRY(cudaEventRecord(ev_done, s->compute));
            return TSB_OK;
          });
          moved = true;
        }
      }
      progress = progress || moved;
    }
    if (status != TSB_OK) break;
    if (finished < static_cast<size_t>(n)) {
      const double t = now();
      if (progress) last_progress = t;
      const bool in_flight = net_busy || !calls.empty() || compute_busy || !release_wait.empty();
      if (!in_flight && next_arrival >= by_arrival.size() && t - last_progress > 5.0) {
        status = fail(TSB_CAPACITY, "stage: no request can make progress (ledger deadlock)");
        break;
      }
      // Nothing to do until the next completion or arrival: back off briefly.
      const double wait = next_arrival < by_arrival.size() ? R[by_arrival[next_arrival]].arrival - t : 1.0;
      if (!progress && wait > 50e-6) {
        timespec ts{0, 20000};
        nanosleep(&ts, nullptr);
      }
    }
  }
  // Drain: no copy thread, ingest or prefill may outlive the call (error paths included).
  {
    const tsb_status ws = worker.drain();
    if (status == TSB_OK) status = ws;
  }
  while (net_busy && !s->net->done()) {
    timespec ts{0, 20000};
    nanosleep(&ts, nullptr);
  }
  cudaStreamSynchronize(st);
  cudaStreamSynchronize(s->compute);
  for (size_t k = 0; k < release_wait.size() && status == TSB_OK; ++k)  // their readers ran (synced)
    status = release_l1(release_wait[k]);
  if (status != TSB_OK) {
    const std::string msg = tsb_last_error();
    for (int64_t i = 0; i < n; ++i) {  // hand every L1 reservation back
      if (!R[i].admitted || R[i].released) continue;
      std::vector<tsb_grant> g(static_cast<size_t>(tsb_l1_deferred(s->l1)) + 1);
      int64_t ng = 0;
      tsb_l1_release_request(s->l1, plans[i].id, g.data(), static_cast<int64_t>(g.size()), &ng);
    }
    return fail(status, msg);
  }

  float last_ms = 0.f;
  for (int64_t i = 0; i < n; ++i) {
    Rt& r = R[i];
    float a = 0.f, b = 0.f, d = 0.f, g = 0.f;
    TSB_CUDA_TRY(cudaEventElapsedTime(&a, s->ev_start, r.ev_first));
    TSB_CUDA_TRY(cudaEventElapsedTime(&b, s->ev_start, r.ev_resident));
    TSB_CUDA_TRY(cudaEventElapsedTime(&d, s->ev_start, r.ev_done));
    TSB_CUDA_TRY(cudaEventElapsedTime(&g, s->ev_start, r.ev_begin));
    last_ms = std::max(last_ms, b);
    if (results)
      results[i] = tsb_stage_request{plans[i].id, pick_pos[i], r.deferred, plans[i].n_chunks,
                                     plans[i].n_chunks * chunk_bytes, a, b, d, r.admit_t * 1e3,
                                     r.arrival * 1e3, g, plans[i].n_chunks * s->shape.chunk_tokens,
                                     plans[i].compute_tokens};
  }
  if (stats) {
    *stats = tsb_stage_stats{};
    stats->bytes = bytes_total;
    stats->device_ms = last_ms;
    stats->wall_ms = (now_s() - wall0) * 1e3;
    stats->ingest_calls = ingest_calls;
    stats->deferred_chunks = deferred_total;
    stats->releases = releases;
    stats->kernel_launches = static_cast<int64_t>(tsb_kernel_launch_count() - launches0);
    stats->verify_mismatches = verify_mismatches;
    stats->net_blocks = net_blocks;
    stats->l2_deferred = l2_deferred;
    stats->reused_chunks = reused_chunks;
  }
  return TSB_OK;
}

}  // extern "C"
