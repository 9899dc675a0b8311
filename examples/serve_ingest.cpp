// serve_ingest.cpp — what a serving engine written against the reference's C++ API does with the
// B200 data plane: plan a batch with the kept API (derive_block_plan), hold the cached chunks in a
// pinned L2 pool (plus, optionally, an HBM tier), lay pages out for the attention backend, and let
// the load stage order, admit and ingest the batch with real bytes.
//
//   g++ -std=c++20 -O2 -Iinclude examples/serve_ingest.cpp -Lpaper_2603_21257_b200 -l:libtsb.so
//       -Wl,-rpath,$PWD/paper_2603_21257_b200 -o serve_ingest
//   ./serve_ingest [requests=4] [ctx_tokens=32768] [policy=lstf] [layout=0|1|2] [tier_chunks=0]
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "tiersim/b200.hpp"
#include "tiersim/cost_model.hpp"
#include "tiersim/scheduler.hpp"
#include "tiersim/types.hpp"

using namespace tiersim;

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 4;
  const std::int64_t ctx = argc > 2 ? std::atoll(argv[2]) : 32768;
  const auto policy = policy_from_name(argc > 3 ? argv[3] : "lstf").value_or(PolicyKind::Lstf);
  const int layout = argc > 4 ? std::atoi(argv[4]) : TSB_LAYOUT_FLASH_ATTN;
  const std::int64_t tier_chunks = argc > 5 ? std::atoll(argv[5]) : 0;
  try {
    KvShape shape;  // Llama-3.1-8B KV: 32 layers, 8 KV heads, d128, bf16, 256-token chunks, 16-token pages
    ClusterConfig cfg;
    cfg.bytes_per_token = kv_bytes_per_token(shape.layers, shape.kv_heads, shape.head_dim, shape.dtype_bytes);
    cfg.block_size_tokens = shape.chunk_tokens;

    // The batch: questions over one long document, with deadlines (LSTF / EDF need them).
    std::vector<RequestSpec> batch;
    for (int i = 0; i < n; ++i) {
      RequestSpec s;
      s.id = 100 + i;
      s.arrival_time = 1e-3 * i;
      s.context_tokens = ctx;
      s.query_tokens = 64;
      s.cache_hit_ratio = 0.9;
      s.deadline = 1.0 + 0.1 * (n - i);
      batch.push_back(s);
    }
    const auto plan = derive_block_plan(batch[0], cfg);  // the reference's chunk plan (types.cpp:85-101)
    const auto nb = static_cast<std::int64_t>(plan.size());

    // L2: the document's chunks in a pinned pool; the first `tier_chunks` also in an HBM tier.
    ChunkPool pool(shape, nb);
    check(tsb_pool_fill_synthetic(pool.handle(), 42, 0, nb, nullptr));
    ChunkPool tier = ChunkPool::on_device(0, shape, nb);
    check(tsb_pool_fill_synthetic(tier.handle(), 42, 0, nb, nullptr));
    std::vector<std::vector<std::int64_t>> slots(static_cast<std::size_t>(n));
    for (auto& s : slots)
      for (std::int64_t c = 0; c < nb; ++c) s.push_back(c < tier_chunks ? ~c : c);

    // L1: room for two requests at a time, so admission defers and releases grant (FIFO).
    PagedAllocator l1(0, shape, 2 * nb * (shape.chunk_tokens / shape.page_tokens), n, nb, nullptr, layout);
    LoadStage stage(l1, pool);
    if (tier_chunks > 0) stage.set_hbm_tier(&tier);
    tsb_stage_options opt{};
    opt.mode = TSB_INGEST_AUTO;
    opt.policy = static_cast<std::int32_t>(policy);
    opt.layer_events = 1;
    opt.verify_seed = 42;
    const auto r = stage.run(batch, slots, cfg, cost_models_from_config(cfg), opt);

    std::printf("%d requests x %lld chunks (%s, layout %d, %lld tier chunks each)\n", n,
                static_cast<long long>(nb), std::string(policy_name(policy)).c_str(), layout,
                static_cast<long long>(tier_chunks));
    for (const auto& q : r.requests)
      std::printf("  request %lld: pick %d, deferred %d, first layer %.1f ms, resident %.1f ms\n",
                  static_cast<long long>(q.request_id), q.pick_position, q.deferred_chunks, q.first_layer_ms,
                  q.resident_ms);
    std::printf("moved %.2f GB in %.1f ms: %.2f GB/s; %lld deferrals, %llu mismatching words\n",
                r.stats.bytes / 1e9, r.stats.device_ms, r.stats.bytes / (r.stats.device_ms * 1e-3) / 1e9,
                static_cast<long long>(r.stats.deferred_chunks),
                static_cast<unsigned long long>(r.stats.verify_mismatches));
    return r.stats.verify_mismatches == 0 ? 0 : 1;
  } catch (const Error& e) {  // the reference's exception classes (error.hpp)
    std::fprintf(stderr, "tiersim error: %s\n", e.what());
    return 2;
  }
}
