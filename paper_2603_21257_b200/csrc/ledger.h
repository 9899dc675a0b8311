// ledger.h — the TierLedger byte ledger (engine.hpp:22-53, engine.cpp:18-49), shared by the
// standalone C-ABI ledger (tsb_ledger_*) and the L1 paged allocator (tsb_l1_*).
#pragma once

#include <stdint.h>

#include <deque>
#include <string>

#include "tsb_capi.h"

namespace tsb {

class Ledger {
 public:
  struct Pending {
    int64_t request_id;
    int32_t block_index;
    int64_t bytes;
  };

  // tier: 0 L3, 1 L2, 2 L1 (types.hpp:20), used only in error text like tier_name().
  Ledger(int tier, int64_t capacity) : tier_(tier), capacity_(capacity) {}

  static const char* tier_name(int tier) {
    return tier == 0 ? "l3" : tier == 1 ? "l2" : tier == 2 ? "l1" : "?";
  }

  // engine.cpp:22-36.  Returns TSB_OK with *granted set, or an error status; msg gets the
  // reference's message text.
  tsb_status request(int64_t request_id, int32_t block_index, int64_t bytes, bool* granted,
                     std::string* msg) {
    if (bytes <= 0) {
      *msg = "TierLedger: reservation bytes must be > 0";
      return TSB_VALIDATION;
    }
    if (bytes > capacity_) {
      *msg = std::string(tier_name(tier_)) + ": reservation of " + std::to_string(bytes) +
             " bytes exceeds capacity " + std::to_string(capacity_);
      return TSB_CAPACITY;
    }
    // Granting past a waiting reservation would starve it; keep strict FIFO.
    if (deferred_.empty() && reserved_ + bytes <= capacity_) {
      reserved_ += bytes;
      *granted = true;
      return TSB_OK;
    }
    deferred_.push_back({request_id, block_index, bytes});
    *granted = false;
    return TSB_OK;
  }

  // engine.cpp:38-49: returns bytes, then grants the waiting queue FIFO while it fits;
  // on_grant(const Pending&) is called for each grant in order.
  template <typename F>
  tsb_status release(int64_t bytes, F&& on_grant, std::string* msg) {
    if (bytes < 0 || bytes > reserved_) {
      *msg = "TierLedger: releasing more than reserved";
      return TSB_VALIDATION;
    }
    reserved_ -= bytes;
    while (!deferred_.empty() && reserved_ + deferred_.front().bytes <= capacity_) {
      const Pending p = deferred_.front();
      reserved_ += p.bytes;
      deferred_.pop_front();
      on_grant(p);
    }
    return TSB_OK;
  }

  int tier() const { return tier_; }
  int64_t capacity() const { return capacity_; }
  int64_t reserved() const { return reserved_; }
  int64_t deferred() const { return static_cast<int64_t>(deferred_.size()); }

 private:
  int tier_;
  int64_t capacity_;
  int64_t reserved_ = 0;
  std::deque<Pending> deferred_;
};

}  // namespace tsb
