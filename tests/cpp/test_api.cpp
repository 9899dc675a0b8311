// C++ drop-in check: reference-style cases written against the kept tiersim C++ API
// (include/tiersim/*.hpp over libtsb.so).  `test_api` runs the host cases; `test_api --gpu`
// adds the cases that need a B200 (scorer/order, ingest, load stage, hasher).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "tiersim/b200.hpp"
#include "tiersim/cost_model.hpp"
#include "tiersim/engine.hpp"
#include "tiersim/scheduler.hpp"
#include "tiersim/types.hpp"
#include "tiersim/workload.hpp"

using namespace tiersim;

static int g_fail = 0, g_run = 0;
#define EXPECT(cond)                                                          \
  do {                                                                        \
    if (!(cond)) {                                                            \
      std::printf("  FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);           \
      ++g_fail;                                                               \
    }                                                                         \
  } while (0)
#define EXPECT_THROW(expr, type)                                              \
  do {                                                                        \
    bool caught = false;                                                      \
    try {                                                                     \
      (void)(expr);                                                           \
    } catch (const type&) {                                                   \
      caught = true;                                                          \
    }                                                                         \
    if (!caught) {                                                            \
      std::printf("  FAIL %s:%d  no %s from %s\n", __FILE__, __LINE__, #type, #expr); \
      ++g_fail;                                                               \
    }                                                                         \
  } while (0)

static void run(const char* name, const std::function<void()>& fn) {
  ++g_run;
  const int before = g_fail;
  try {
    fn();
  } catch (const std::exception& e) {
    std::printf("  FAIL %s: exception %s\n", name, e.what());
    ++g_fail;
  }
  std::printf("%s %s\n", g_fail == before ? "ok  " : "FAIL", name);
}

static RequestSpec spec(std::int64_t id, double arrival, std::int64_t ctx, std::int64_t query = 10,
                        double hit = 1.0) {
  RequestSpec s;
  s.id = id;
  s.arrival_time = arrival;
  s.context_tokens = ctx;
  s.query_tokens = query;
  s.cache_hit_ratio = hit;
  return s;
}

static std::vector<std::int64_t> drain(std::vector<RequestSpec> q, PolicyKind p, const CostMap& c) {
  std::vector<std::int64_t> out;
  while (auto r = pick_next(q, p, c, 0.0)) out.push_back(r->id);
  return out;
}

static void host_cases() {
  run("plan: floor rule and whole blocks", [] {
    const ClusterConfig cfg;
    EXPECT(derive_block_plan(spec(1, 0, 512), cfg).size() == 2);
    const auto p = derive_block_plan(spec(2, 0, 28100), cfg);
    EXPECT(p.size() == 109 && p.back().block_index == 108 && p[0].bytes == 256 * 131072);
    EXPECT(cached_token_count(spec(2, 0, 28100), cfg) == 27904);
    EXPECT(derive_block_plan(spec(3, 0, 28100, 10, 0.0), cfg).empty());
    const auto st = make_request_state(spec(4, 1.5, 1000, 7, 0.5), cfg);
    EXPECT(st.cached_tokens == 256 && st.compute_tokens == 1000 + 7 - 256 && st.ts.arrival == 1.5);
  });
  run("events: names and the reference CSV layout", [] {
    EXPECT(std::string(stage_name(Stage::Pcie)) == "pcie" && std::string(event_kind_name(EventKind::DispatchWake)) == "dispatch_wake");
    tsb_trace_row row{0.5, 3, 2, -1, 2, 7, 11, 4096};
    const TraceEvent e = trace_event_of(row);
    EXPECT(e.kind == EventKind::AllocationGrant && !e.stage && e.tier == Tier::L1 && e.block_index == 7);
    const auto csv = std::filesystem::temp_directory_path() / "tsb_events_test.csv";
    write_trace_csv(csv, std::vector<TraceEvent>{e});
    std::ifstream in(csv);
    std::string a, b;
    std::getline(in, a);
    std::getline(in, b);
    EXPECT(b == "0.500000000,3,allocation_grant,l1,11,7,4096");
    std::filesystem::remove(csv);
  });
  run("config_fingerprint: reference golden (tests/golden/ref_misc.json)", [] {
    ClusterConfig cfg;
    EXPECT(config_fingerprint(cfg, PolicyKind::Fifo, 0) == 18430105898594341330ull);
    cfg.pcie_bandwidth = 55.6e9;
    EXPECT(config_fingerprint(cfg, PolicyKind::Lstf, 7) == 12797939754527448084ull);
  });
  run("workload: generate_workload / assign_slos through the kept API", [] {
    WorkloadSpec w;
    w.profile = builtin_profile("loogle");
    w.count = 500;
    w.qps = 4.0;
    w.seed = 9;
    w.hit_ratio_source = HitRatioSource::uniform_choice({0.25, 0.5, 1.0});
    const auto a = generate_workload(w), b = generate_workload(w);
    EXPECT(a.size() == 500 && a.front().id == 1 && a.back().id == 500 && a[0].dataset_tag == "loogle");
    bool ok = true;
    for (std::size_t i = 0; i < a.size(); ++i) {
      ok = ok && a[i].context_tokens == b[i].context_tokens && a[i].arrival_time == b[i].arrival_time;
      ok = ok && a[i].context_tokens >= 1 && a[i].query_tokens >= 1;
      ok = ok && (i == 0 || a[i].arrival_time - a[i - 1].arrival_time >= 1e-6 * 0.999999);
      ok = ok && (a[i].cache_hit_ratio == 0.25 || a[i].cache_hit_ratio == 0.5 || a[i].cache_hit_ratio == 1.0);
    }
    EXPECT(ok);
    ClusterConfig cfg;
    cfg.l1_capacity = cfg.l2_capacity = 10'000'000'000'000;
    const std::vector<double> f = {2.0, 4.0, 8.0};
    const auto s = assign_slos(a, cfg, cost_models_from_config(cfg), f, 3);
    bool dl = true;
    for (std::size_t i = 0; i < s.size(); ++i) {
      const double solo = solo_baseline_ttft(a[i], cfg);
      const double fac = (*s[i].deadline - a[i].arrival_time) / solo;
      dl = dl && s[i].deadline.has_value() && fac > 1.99 && fac < 8.01;
    }
    EXPECT(dl);
    bool threw = false;
    try {
      builtin_profile("nope");
    } catch (const UnknownProfile&) {
      threw = true;
    }
    EXPECT(threw);
  });
  run("geometry: kv_bytes_per_token", [] {
    EXPECT(kv_bytes_per_token(32, 8, 128, 2) == 131072);
    EXPECT(kv_bytes_per_token(64, 8, 128, 2) == 262144);
    EXPECT_THROW(kv_bytes_per_token(0, 8, 128, 2), ValidationError);
  });
  run("validation messages", [] {
    RequestSpec s = spec(9, 2.0, 10);
    s.deadline = 1.0;
    EXPECT_THROW(s.validate(), ValidationError);
    s = spec(9, 0, 10, 0);
    EXPECT_THROW(s.validate(), ValidationError);
    ClusterConfig c;
    c.pcie_bandwidth = 0;
    EXPECT_THROW(c.validate(), ValidationError);
  });
  run("cost model: predict, overrides, cache miss, config models", [] {
    EXPECT(std::fabs(predict({1e-4, 0.1}, 2610) - 0.361) < 1e-12);
    RequestSpec s = spec(1, 0, 1000);
    s.measured_cost = MeasuredCost{0.361, 0.019};
    const ClusterConfig cfg;
    const auto c = estimate_service_cost(s, {1e-5, 0}, {1e-5, 0}, cfg);
    EXPECT(c.t_load == 0.361 && c.t_comp == 0.019);
    const auto miss = estimate_service_cost(spec(2, 0, 5000, 100, 0.0), {1e-4, 0}, {1e-5, 0.01}, cfg);
    EXPECT(miss.t_load == 0.0 && miss.t_comp > 0.0);
    const auto m = cost_models_from_config(cfg);
    const double block = 256.0 * 131072.0;
    const double want = 2 * cfg.transfer_base_latency + block / cfg.network_bandwidth + block / cfg.pcie_bandwidth;
    EXPECT(std::fabs(predict(m.load, 256) - want) < 1e-12 * want);
    EXPECT(m.comp.intercept == cfg.compute_base && m.comp.slope == cfg.compute_per_token);
  });
  run("fit_linear: exact, degenerate, clamped; samples CSV", [] {
    std::vector<TokenSample> s = {{0, 0.1}, {1000, 0.2}, {3000, 0.4}};
    const auto f = fit_linear(s);
    EXPECT(std::fabs(f.model.slope - 1e-4) < 1e-15 && std::fabs(f.model.intercept - 0.1) < 1e-12);
    std::vector<TokenSample> one = {{5, 0.1}, {5, 0.2}};
    EXPECT_THROW(fit_linear(one), DegenerateFit);
    std::vector<TokenSample> fall = {{0, 0.5}, {1000, 0.1}};
    EXPECT(fit_linear(fall).slope_clamped);
    const auto p = std::filesystem::temp_directory_path() / "tsb_samples.csv";
    std::ofstream(p) << "tokens,seconds\n# ingest calibration\n256,0.0047\n512,0.0093\n";
    const auto rows = read_samples_csv(p);
    EXPECT(rows.size() == 2 && rows[1].tokens == 512);
  });
  run("ledger: exact fit, FIFO deferral without bypass, errors", [] {
    TierLedger a(Tier::L1, 100);
    EXPECT(a.request(1, 0, 40) == TierLedger::Outcome::Granted);
    EXPECT(a.request(1, 1, 60) == TierLedger::Outcome::Granted && a.reserved() == 100);
    TierLedger b(Tier::L1, 100);
    EXPECT(b.request(1, 0, 90) == TierLedger::Outcome::Granted);
    EXPECT(b.request(2, 0, 20) == TierLedger::Outcome::Deferred);
    EXPECT(b.request(3, 0, 5) == TierLedger::Outcome::Deferred && b.deferred_count() == 2);
    const auto g = b.release(20);
    EXPECT(g.size() == 2 && g[0].request_id == 2 && g[1].request_id == 3 && b.reserved() == 95);
    TierLedger c(Tier::L2, 100);
    EXPECT_THROW(c.request(1, 0, 101), CapacityError);
    EXPECT_THROW(c.request(1, 0, 0), ValidationError);
    EXPECT_THROW(c.release(1), ValidationError);
  });
  run("policies: names, keys, missing deadline", [] {
    for (PolicyKind p : all_policies()) EXPECT(policy_from_name(policy_name(p)) == p);
    EXPECT(!policy_from_name("sjf"));
    RequestSpec s = spec(5, 0, 1000, 10, 0.5);
    EXPECT(prefill_token_estimate(s) == 1010.0 - 500.0);
    EXPECT_THROW(priority_key(s, PolicyKind::Lstf, ServiceCost{}, 0.0), MissingDeadline);
    s.deadline = 2.0;
    const auto k = priority_key(s, PolicyKind::Lstf, ServiceCost{0.5, 0.25}, 0.0);
    EXPECT(k.primary == 2.0 - 0.75 && k.id == 5);
  });
}

static void gpu_cases() {
  run("gpu: pick_next drain (SJF-cost vs FIFO, LSTF vs EDF, tie-breaks)", [] {
    CostMap costs{{1, {0.361, 0.019}}, {2, {0.199, 0.025}}};
    const std::vector<RequestSpec> q = {spec(1, 0, 1000), spec(2, 0, 1000)};
    EXPECT((drain(q, PolicyKind::SjfCost, costs) == std::vector<std::int64_t>{2, 1}));
    EXPECT((drain(q, PolicyKind::Fifo, costs) == std::vector<std::int64_t>{1, 2}));
    RequestSpec a = spec(1, 0, 1000), b = spec(2, 0, 1000);
    a.deadline = 1.0;
    b.deadline = 0.8;
    CostMap c2{{1, {0.4, 0.1}}, {2, {0.05, 0.05}}};
    EXPECT((drain({a, b}, PolicyKind::Lstf, c2) == std::vector<std::int64_t>{1, 2}));
    EXPECT((drain({a, b}, PolicyKind::Edf, c2) == std::vector<std::int64_t>{2, 1}));
    CostMap c3{{7, {0.1, 0.1}}, {9, {0.1, 0.1}}, {11, {0.1, 0.1}}};
    EXPECT((drain({spec(11, 1, 1000), spec(7, 1, 1000), spec(9, 1, 1000)}, PolicyKind::SjfCost, c3) ==
            std::vector<std::int64_t>{7, 9, 11}));
    EXPECT((schedule_order(std::vector<RequestSpec>{spec(7, 2, 1000), spec(9, 1, 1000)}, PolicyKind::SjfCost, c3) ==
            std::vector<std::int64_t>{9, 7}));
    EXPECT_THROW(drain({spec(1, 0, 10), b}, PolicyKind::Edf, {}), MissingDeadline);
  });
  run("gpu: load stage under L1 pressure", [] {
    KvShape shape;
    shape.layers = 4;
    ChunkPool pool(shape, 8);
    check(tsb_pool_fill_synthetic(pool.handle(), 99, 0, 8, nullptr));
    PagedAllocator l1(0, shape, 6 * 16, 8, 8);
    LoadStage stage(l1, pool);
    ClusterConfig cfg;
    cfg.bytes_per_token = kv_bytes_per_token(4, 8, 128, 2);
    std::vector<RequestSpec> batch = {spec(1, 0.0, 256 * 5), spec(2, 0.1, 256 * 4), spec(3, 0.2, 256 * 5)};
    std::vector<std::vector<int64_t>> slots = {{0, 1, 2, 3, 4}, {4, 5, 6, 7}, {3, 2, 1, 0, 7}};
    tsb_stage_options opt{};
    opt.mode = TSB_INGEST_AUTO;
    opt.policy = static_cast<int32_t>(PolicyKind::Fifo);
    opt.verify_seed = 99;
    const auto r = stage.run(batch, slots, cfg, cost_models_from_config(cfg), opt);
    EXPECT(r.stats.verify_mismatches == 0 && r.stats.deferred_chunks > 0 && l1.reserved() == 0);
    EXPECT(r.stats.bytes == 14 * 256 * cfg.bytes_per_token);
  });
  run("gpu: load stage from a device-resident (peer-HBM tier) pool", [] {
    KvShape shape;
    shape.layers = 4;
    ChunkPool pool = ChunkPool::on_device(0, shape, 8);
    EXPECT(pool.on_device());
    check(tsb_pool_fill_synthetic(pool.handle(), 41, 0, 8, nullptr));
    PagedAllocator l1(0, shape, 6 * 16, 8, 8);
    LoadStage stage(l1, pool);
    ClusterConfig cfg;
    cfg.bytes_per_token = kv_bytes_per_token(4, 8, 128, 2);
    std::vector<RequestSpec> batch = {spec(1, 0.0, 256 * 5), spec(2, 0.1, 256 * 4)};
    std::vector<std::vector<int64_t>> slots = {{0, 1, 2, 3, 4}, {4, 5, 6, 7}};
    tsb_stage_options opt{};
    opt.mode = TSB_INGEST_AUTO;
    opt.verify_seed = 41;
    const auto r = stage.run(batch, slots, cfg, cost_models_from_config(cfg), opt);
    EXPECT(r.stats.verify_mismatches == 0 && r.stats.deferred_chunks > 0 && l1.reserved() == 0);
    unsigned char h[64];
    pool.ipc_handle(h);  // exportable to the other per-GPU processes
  });
  run("gpu: load stage with an HBM tier and FlashInfer HND pages", [] {
    KvShape shape;
    shape.layers = 4;
    ChunkPool pool(shape, 8);
    check(tsb_pool_fill_synthetic(pool.handle(), 77, 0, 8, nullptr));
    ChunkPool tier = ChunkPool::on_device(0, shape, 8);
    check(tsb_pool_fill_synthetic(tier.handle(), 77, 0, 8, nullptr));  // same content per slot
    PagedAllocator l1(0, shape, 6 * 16, 8, 8, nullptr, TSB_LAYOUT_FLASHINFER_HND);
    EXPECT(l1.layout() == TSB_LAYOUT_FLASHINFER_HND);
    LoadStage stage(l1, pool);
    stage.set_hbm_tier(&tier);
    ClusterConfig cfg;
    cfg.bytes_per_token = kv_bytes_per_token(4, 8, 128, 2);
    std::vector<RequestSpec> batch = {spec(1, 0.0, 256 * 5), spec(2, 0.1, 256 * 4)};
    std::vector<std::vector<int64_t>> slots = {{~0ll, ~1ll, 2, 3, 4}, {4, ~5ll, 6, ~7ll}};  // ~s: HBM tier
    tsb_stage_options opt{};
    opt.mode = TSB_INGEST_AUTO;
    opt.verify_seed = 77;
    const auto r = stage.run(batch, slots, cfg, cost_models_from_config(cfg), opt);
    EXPECT(r.stats.verify_mismatches == 0 && r.stats.deferred_chunks > 0 && l1.reserved() == 0);
    EXPECT(r.stats.bytes == 9 * 256 * cfg.bytes_per_token);
    // one item-layer per copy-engine group (the knob the stage sets itself under a prefill)
    l1.set_ce_group_bytes(2 * 256 * 8 * 128 * 2);
    EXPECT(l1.ce_group_bytes() == 2 * 256 * 8 * 128 * 2);
    opt.mode = TSB_INGEST_CE;
    opt.verify_seed = 77;  // the pools hold seed 77
    const auto r2 = stage.run(batch, slots, cfg, cost_models_from_config(cfg), opt);
    EXPECT(r2.stats.verify_mismatches == 0 && l1.reserved() == 0);
  });
  run("gpu: pick_next drain == schedule_order, keys computed once per request", [] {
    std::vector<RequestSpec> q;
    for (int i = 0; i < 300; ++i) {
      RequestSpec r = spec(1000 + i, 0.001 * ((i * 37) % 300), 256 * (1 + (i * 13) % 40));
      r.cache_hit_ratio = (i % 3) ? 0.9 : 0.5;
      r.deadline = r.arrival_time + 1.0 + 0.01 * (i % 17);
      q.push_back(r);
    }
    CostMap costs;
    for (int i = 0; i < 300; i += 3) costs[1000 + i] = ServiceCost{0.001 * (i % 7), 0.002};
    for (PolicyKind p : {PolicyKind::Lstf, PolicyKind::SjfCost}) {
      const auto want = schedule_order(q, p, costs);
      std::vector<RequestSpec> work = q;
      const uint64_t l0 = tsb_kernel_launch_count();
      std::vector<std::int64_t> got;
      while (auto r = pick_next(work, p, costs, 0.0)) got.push_back(r->id);
      const uint64_t launches = tsb_kernel_launch_count() - l0;
      EXPECT(got == want);
      EXPECT(launches < 20);  // one scoring pass for the whole drain, not 300
      // a new arrival is scored on its own and slots into the cached order
      work = q;
      RequestSpec late = spec(5000, 0.0, 256);
      late.deadline = 0.01;
      work.push_back(late);
      const auto first = pick_next(work, p, costs, 0.0);
      EXPECT(first && (p != PolicyKind::Lstf || first->id == 5000));
    }
  });
  run("gpu: online stage with an L3 store, coupled + reactive, a C prefill hook", [] {
    KvShape shape;
    shape.layers = 4;
    ChunkPool l3(shape, 12), l2(shape, 6);
    check(tsb_pool_fill_synthetic(l3.handle(), 55, 0, 12, nullptr));
    check(tsb_pool_fill_synthetic(l2.handle(), 1, 0, 6, nullptr));
    PagedAllocator l1(0, shape, 8 * 16, 8, 8);
    LoadStage stage(l1, l2);
    stage.set_l3(&l3, 2);
    static int calls = 0;
    calls = 0;
    stage.set_prefill_hook([](void*, int64_t, int32_t, int64_t, void*) -> int { return ++calls > 0 ? 0 : 1; }, nullptr);
    ClusterConfig cfg;
    cfg.bytes_per_token = kv_bytes_per_token(4, 8, 128, 2);
    cfg.l2_capacity = 6 * 256 * cfg.bytes_per_token;
    cfg.control_mode = ControlMode::Coupled;
    cfg.allocation_mode = AllocationMode::Reactive;
    std::vector<RequestSpec> batch = {spec(1, 0.0, 256 * 5), spec(2, 0.001, 256 * 4), spec(3, 0.002, 256 * 6)};
    std::vector<std::vector<int64_t>> slots = {{0, 1, 2, 3, 4}, {7, 8, 9, 10}, {11, 5, 6, 0, 1, 2}};
    tsb_stage_options opt{};
    opt.mode = TSB_INGEST_AUTO;
    opt.prefill = 1;
    opt.verify_seed = 55;
    opt.record_trace = 1;
    const auto r = stage.run_online(batch, slots, cfg, cost_models_from_config(cfg), opt);
    EXPECT(r.stats.verify_mismatches == 0 && r.stats.net_blocks == 15 && l1.reserved() == 0);
    EXPECT(calls == 3 * 4);  // every layer of every request went through the hook
    // the TraceEvent stream (events.hpp): per block one L2 and one L1 grant, one net and one pcie
    // hop, each dispatched after its grant (trace_checks.hpp:93-143); one compute_done per request
    const std::vector<TraceEvent> tr = stage.trace();
    std::map<std::pair<int64_t, int32_t>, std::uint64_t> g1, g2, net, pcie, done;
    int computes = 0;
    for (const TraceEvent& e : tr) {
      const auto key = std::make_pair(e.request_id, e.block_index);
      if (e.kind == EventKind::AllocationGrant) (*e.tier == Tier::L1 ? g1 : g2)[key] = e.seq;
      if (e.kind == EventKind::DispatchWake && e.stage == Stage::Net) {
        EXPECT(g2.count(key) && g2[key] < e.seq && !net.count(key));
        net[key] = e.seq;
      }
      if (e.kind == EventKind::DispatchWake && e.stage == Stage::Pcie) {
        EXPECT(g1.count(key) && g1[key] < e.seq && !pcie.count(key));
        pcie[key] = e.seq;
      }
      if (e.kind == EventKind::TransferDone && e.stage == Stage::Pcie) done[key] = e.seq;
      if (e.kind == EventKind::ComputeDone) ++computes;
    }
    EXPECT(g1.size() == 15 && g2.size() == 15 && net.size() == 15 && pcie.size() == 15 && done.size() == 15);
    EXPECT(computes == 3);
    const auto csv = std::filesystem::temp_directory_path() / "tsb_trace_test.csv";
    write_trace_csv(csv, tr);
    std::ifstream in(csv);
    std::string line;
    std::getline(in, line);
    EXPECT(line == "time,seq,kind,stage,request_id,block_index,bytes");
    std::size_t rows = 0;
    while (std::getline(in, line)) ++rows;
    EXPECT(rows == tr.size());
    std::filesystem::remove(csv);
  });
  run("gpu: prefix hasher", [] {
    std::vector<std::int64_t> off = {0, 600, 1112};
    std::vector<std::int32_t> tok(1112);
    for (std::size_t i = 0; i < tok.size(); ++i) tok[i] = static_cast<std::int32_t>(i % 600);
    const auto h = hash_prefix_chunks(off, tok);
    EXPECT(h.size() == 2 + 2 && h[0] == h[2] && h[1] == h[3]);  // identical 512-token prefixes
  });
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
  host_cases();
  if (gpu) gpu_cases();
  std::printf("%d cases, %d failures\n", g_run, g_fail);
  return g_fail ? 1 : 0;
}
