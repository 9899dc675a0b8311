// tiersim/engine.hpp — TierLedger of the reference (core/include/tiersim/engine.hpp:22-53), backed by
// libtsb's tsb::Ledger: identical grant/defer decisions, FIFO grant lists and error messages.
// The L1 tier with real pages is tiersim::PagedAllocator (tiersim/b200.hpp), which runs the same
// ledger, and config_fingerprint.  run_simulation (the DES) is out of scope: the real-time path is
// tiersim::LoadStage.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "tiersim/error.hpp"
#include "tiersim/scheduler.hpp"
#include "tiersim/types.hpp"

namespace tiersim {

class TierLedger {
 public:
  enum class Outcome : std::uint8_t { Granted, Deferred };
  struct Pending {
    std::int64_t request_id = 0;
    std::int32_t block_index = 0;
    std::int64_t bytes = 0;
  };

  TierLedger(Tier tier, std::int64_t capacity) : tier_(tier) {
    tsb_ledger* l = nullptr;
    check(tsb_ledger_create(static_cast<int>(tier), capacity, &l));
    l_.reset(l);
  }

  Outcome request(std::int64_t request_id, std::int32_t block_index, std::int64_t bytes) {
    int granted = 0;
    check(tsb_ledger_request(l_.get(), request_id, block_index, bytes, &granted));
    return granted ? Outcome::Granted : Outcome::Deferred;
  }

  std::vector<Pending> release(std::int64_t bytes) {
    std::vector<tsb_grant> g(static_cast<std::size_t>(deferred_count()) + 1);
    int64_t n = 0;
    check(tsb_ledger_release(l_.get(), bytes, g.data(), static_cast<int64_t>(g.size()), &n));
    std::vector<Pending> out(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) out[i] = {g[i].request_id, g[i].block_index, g[i].bytes};
    return out;
  }

  Tier tier() const noexcept { return tier_; }
  std::int64_t capacity() const noexcept { return tsb_ledger_capacity(l_.get()); }
  std::int64_t reserved() const noexcept { return tsb_ledger_reserved(l_.get()); }
  std::size_t deferred_count() const noexcept {
    return static_cast<std::size_t>(tsb_ledger_deferred(l_.get()));
  }

 private:
  struct Del {
    void operator()(tsb_ledger* l) const { tsb_ledger_destroy(l); }
  };
  Tier tier_;
  std::unique_ptr<tsb_ledger, Del> l_;
};

// config_fingerprint (engine.hpp:68-74): FNV-1a-64 of the config, policy and seed.
inline std::uint64_t config_fingerprint(const ClusterConfig& config, PolicyKind policy, std::uint64_t seed) {
  const tsb_cluster c = config.c_abi();
  return tsb_config_fingerprint(&c, static_cast<int>(policy), seed);
}

}  // namespace tiersim
