// tiersim/events.hpp — the reference's TraceEvent schema (core/include/tiersim/events.hpp:17-46),
// the observable contract of its load stage.  LoadStage::trace() returns the
// rows of the last real-time run (record_trace set) in this schema, so the reference's trace
// checks (proj/tests/trace_checks.hpp) and its CSV writer apply to real runs unchanged.
#pragma once

#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <optional>
#include <span>
#include <vector>

#include "tiersim/error.hpp"
#include "tiersim/types.hpp"
#include "tsb_capi.h"

namespace tiersim {

enum class Stage : std::uint8_t { Net, Pcie, Compute };

inline const char* stage_name(Stage stage) {
  switch (stage) {
    case Stage::Net: return "net";
    case Stage::Pcie: return "pcie";
    case Stage::Compute: return "compute";
  }
  return "?";
}

enum class EventKind : std::uint8_t { Arrival, TransferDone, AllocationGrant, ComputeDone, DispatchWake };

inline const char* event_kind_name(EventKind kind) {
  switch (kind) {
    case EventKind::Arrival: return "arrival";
    case EventKind::TransferDone: return "transfer_done";
    case EventKind::AllocationGrant: return "allocation_grant";
    case EventKind::ComputeDone: return "compute_done";
    case EventKind::DispatchWake: return "dispatch_wake";
  }
  return "?";
}

struct TraceEvent {
  double time = 0.0;
  std::uint64_t seq = 0;
  EventKind kind = EventKind::Arrival;
  std::optional<Stage> stage;  // TransferDone / ComputeDone / DispatchWake
  std::optional<Tier> tier;    // AllocationGrant
  std::int64_t request_id = -1;
  std::int32_t block_index = -1;
  std::int64_t bytes = 0;
};

/// One C-ABI trace row (stage / tier < 0 = unset) as a TraceEvent.
inline TraceEvent trace_event_of(const tsb_trace_row& r) {
  TraceEvent e;
  e.time = r.time;
  e.seq = r.seq;
  e.kind = static_cast<EventKind>(r.kind);
  if (r.stage >= 0) e.stage = static_cast<Stage>(r.stage);
  if (r.tier >= 0) e.tier = static_cast<Tier>(r.tier);
  e.request_id = r.request_id;
  e.block_index = r.block_index;
  e.bytes = r.bytes;
  return e;
}

/// CSV with columns (time, seq, kind, stage, request_id, block_index, bytes); the stage column
/// carries the tier name for allocation grants (events.cpp:33-47).
inline void write_trace_csv(const std::filesystem::path& path, std::span<const TraceEvent> trace) {
  std::ofstream out(path);
  if (!out) throw Error("write_trace_csv: cannot open " + path.string());
  out << "time,seq,kind,stage,request_id,block_index,bytes\n";
  char t[64];
  for (const TraceEvent& ev : trace) {
    std::snprintf(t, sizeof(t), "%.9f", ev.time);
    out << t << ',' << ev.seq << ',' << event_kind_name(ev.kind) << ',';
    if (ev.stage) out << stage_name(*ev.stage);
    else if (ev.tier) out << tier_name(*ev.tier);
    out << ',' << ev.request_id << ',' << ev.block_index << ',' << ev.bytes << '\n';
  }
}

}  // namespace tiersim
