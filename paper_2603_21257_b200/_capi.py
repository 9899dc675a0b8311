"""ctypes binding of libtsb.so (include/tsb_capi.h).

This is the reference-side binding a Python caller would add (INTEGRATION.md shows the same
declarations); every higher-level module in the package goes through it.  There is no
fallback: importing the package without the built library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("TSB_LIB", _HERE / "libtsb.so"))

if not LIB_PATH.exists():
    raise ImportError(
        f"libtsb.so not found at {LIB_PATH}: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "or `make -C paper_2603_21257_b200` (no CPU fallback exists)."
    )

lib = C.CDLL(str(LIB_PATH))

# ---- status -------------------------------------------------------------------------------
(TSB_OK, TSB_VALIDATION, TSB_CAPACITY, TSB_MISSING_DEADLINE, TSB_DEGENERATE_FIT, TSB_CUDA, TSB_UNSUPPORTED,
 TSB_UNKNOWN_PROFILE) = range(8)

i64, u64, f64, i32, u8 = C.c_int64, C.c_uint64, C.c_double, C.c_int32, C.c_uint8
P = C.POINTER
vp = C.c_void_p


class Cluster(C.Structure):
    """tsb_cluster == tiersim::ClusterConfig (types.hpp:82-97)."""

    _fields_ = [
        ("network_bandwidth", f64),
        ("pcie_bandwidth", f64),
        ("transfer_base_latency", f64),
        ("l1_capacity", i64),
        ("l2_capacity", i64),
        ("bytes_per_token", i64),
        ("block_size_tokens", i64),
        ("compute_base", f64),
        ("compute_per_token", f64),
        ("compute_quadratic", f64),
        ("allocation_mode", i32),
        ("control_mode", i32),
    ]


class KvShape(C.Structure):
    _fields_ = [
        ("layers", i64),
        ("kv_heads", i64),
        ("head_dim", i64),
        ("dtype_bytes", i64),
        ("chunk_tokens", i64),
        ("page_tokens", i64),
        ("tp_size", i64),
        ("tp_rank", i64),
    ]


class Queue(C.Structure):
    """tsb_queue: struct-of-arrays RequestSpec queue (pointers may be host or device)."""

    _fields_ = [
        ("id", vp),
        ("arrival", vp),
        ("context_tokens", vp),
        ("query_tokens", vp),
        ("cache_hit_ratio", vp),
        ("flags", vp),
        ("deadline", vp),
        ("measured_t_load", vp),
        ("measured_t_comp", vp),
    ]


class WorkloadSpec(C.Structure):
    """tsb_workload_spec == DatasetProfile + WorkloadSpec (workload.hpp:19-68)."""

    _fields_ = [("num_requests", i64), ("context_tokens_mean", f64), ("context_tokens_cv", f64),
                ("query_tokens_mean", f64), ("query_tokens_cv", f64), ("qps", f64), ("count", i64),
                ("hit_kind", i32), ("hit_fixed", f64), ("hit_choices", vp), ("n_hit_choices", i64),
                ("seed", u64)]


class Grant(C.Structure):
    _fields_ = [("request_id", i64), ("block_index", i32), ("bt_row", i32), ("bytes", i64)]


class IngestItem(C.Structure):
    _fields_ = [("src_slot", i64), ("bt_row", i32), ("chunk_index", i32)]


class StageOptions(C.Structure):
    _fields_ = [("mode", i32), ("policy", i32), ("layer_events", i32), ("prefill", i32), ("prefill_ctas", i32),
                ("record_trace", i32), ("verify_seed", u64), ("pace_network", i32), ("reuse_l1", i32)]


class StageRequest(C.Structure):
    _fields_ = [("request_id", i64), ("pick_position", i32), ("deferred_chunks", i32), ("chunks", i64),
                ("bytes", i64), ("first_layer_ms", f64), ("resident_ms", f64), ("done_ms", f64),
                ("admit_ms", f64), ("arrival_ms", f64), ("ingest_begin_ms", f64), ("cached_tokens", i64),
                ("compute_tokens", i64)]


class StageStats(C.Structure):
    _fields_ = [("bytes", i64), ("device_ms", f64), ("wall_ms", f64), ("ingest_calls", i64),
                ("deferred_chunks", i64), ("releases", i64), ("kernel_launches", i64), ("verify_mismatches", u64),
                ("net_blocks", i64), ("l2_deferred", i64), ("reused_chunks", i64)]


class TraceRow(C.Structure):
    _fields_ = [("time", f64), ("seq", u64), ("kind", i32), ("stage", i32), ("tier", i32), ("block_index", i32),
                ("request_id", i64), ("bytes", i64)]


HAS_DEADLINE, HAS_MEASURED = 1, 2
INGEST_AUTO, INGEST_ZEROCOPY, INGEST_BULK, INGEST_CE, INGEST_CE_DIRECT = range(5)
POOL_HOST, POOL_DEVICE = 0, 1


def _decl(name, restype, *argtypes):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


st = C.c_int
_decl("tsb_last_error", C.c_char_p)
_decl("tsb_version", C.c_char_p)
_decl("tsb_kernel_launch_count", u64)
_decl("tsb_current_device", C.c_int)
_decl("tsb_cluster_default", None, P(Cluster))
_decl("tsb_cluster_validate", st, P(Cluster))
_decl("tsb_config_fingerprint", u64, P(Cluster), C.c_int, u64)
_decl("tsb_kv_bytes_per_token", st, i64, i64, i64, i64, P(i64))
_decl("tsb_kv_shape_info", st, P(KvShape), P(i64), P(i64), P(i64))
_decl("tsb_request_validate", st, P(Queue), i64)
_decl("tsb_derive_block_plan", st, P(Queue), i64, P(Cluster), P(i64), P(i64), P(i64), P(i64), P(i64))
_decl("tsb_builtin_profile", st, C.c_char_p, P(WorkloadSpec))
_decl("tsb_workload_validate", st, P(WorkloadSpec))
_decl("tsb_workload_count", i64, P(WorkloadSpec))
_decl("tsb_generate_workload", st, P(WorkloadSpec), i64, vp, vp, vp, vp, vp, P(i64))
_decl("tsb_solo_baseline_ttft", st, P(Queue), i64, P(Cluster), P(f64))
_decl("tsb_assign_slos", st, i64, P(Queue), P(Cluster), vp, i64, u64, vp)
_decl("tsb_cost_models_from_config", None, P(Cluster), P(f64))
_decl("tsb_predict", f64, f64, f64, i64)
_decl("tsb_fit_linear", st, i64, vp, vp, P(f64), P(f64), P(C.c_int), P(C.c_int))
_decl("tsb_estimate_service_cost", st, P(Queue), i64, P(f64), P(Cluster), P(f64), P(f64))
_decl("tsb_priority_key", st, P(Queue), i64, C.c_int, f64, f64, P(f64))
_decl("tsb_scorer_create", st, C.c_int, i64, P(vp))
_decl("tsb_scorer_destroy", None, vp)
_decl("tsb_score_queue_device", st, vp, vp, i64, P(Queue), C.c_int, P(f64), P(Cluster), vp, vp, vp, vp, P(i64))
_decl("tsb_scorer_check", st, vp, vp, P(i64))
_decl("tsb_score_queue", st, vp, vp, i64, P(Queue), C.c_int, P(f64), P(Cluster), vp, vp, vp, vp)
_decl("tsb_hash_prefix_chunks_device", st, vp, i64, vp, vp, vp, vp)
_decl("tsb_hash_prefix_chunks", st, vp, i64, vp, vp, vp, P(i64))
_decl("tsb_hash_chunk_digests_device", st, vp, i64, vp, vp, vp, vp)
_decl("tsb_hash_set_grid", st, C.c_int)
_decl("tsb_hash_set_tuning", st, C.c_int, C.c_int)
_decl("tsb_gen_tokens_device", st, vp, u64, i64, vp, vp, vp, vp)
_decl("tsb_index_create", st, C.c_int, i64, P(vp))
_decl("tsb_index_destroy", None, vp)
_decl("tsb_index_capacity", i64, vp)
_decl("tsb_index_insert_device", st, vp, vp, i64, vp, vp)
_decl("tsb_index_erase_device", st, vp, vp, i64, vp)
_decl("tsb_index_lookup_device", st, vp, vp, i64, vp, vp, vp, vp)
_decl("tsb_index_stats", st, vp, vp, P(i64), P(i64))
_decl("tsb_index_insert", st, vp, vp, i64, vp, vp)
_decl("tsb_index_clear", st, vp, vp)
_decl("tsb_index_compact", st, vp, vp, P(i64))
_decl("tsb_index_lookup", st, vp, vp, i64, vp, vp, vp, vp)
_decl("tsb_pool_create", st, P(KvShape), i64, P(vp))
_decl("tsb_pool_wrap", st, P(KvShape), vp, i64, P(vp))
_decl("tsb_pool_register", st, P(KvShape), vp, i64, P(vp))
_decl("tsb_pool_create_numa", st, P(KvShape), i64, C.c_int, P(vp))
_decl("tsb_pool_numa_node", C.c_int, vp)
_decl("tsb_device_numa_node", C.c_int, C.c_int)
_decl("tsb_pool_destroy", None, vp)
_decl("tsb_pool_slot_ptr", vp, vp, i64)
_decl("tsb_pool_slots", i64, vp)
_decl("tsb_pool_chunk_bytes", i64, vp)
_decl("tsb_pool_fill_synthetic", st, vp, u64, i64, i64, vp)
_decl("tsb_pool_create_device", st, C.c_int, P(KvShape), i64, P(vp))
_decl("tsb_pool_wrap_device", st, C.c_int, P(KvShape), vp, i64, P(vp))
_decl("tsb_pool_ipc_handle", st, vp, C.c_char_p)
_decl("tsb_pool_open_ipc", st, P(KvShape), C.c_char_p, C.c_int, i64, P(vp))
_decl("tsb_enable_peer_access", st, C.c_int, C.c_int)
_decl("tsb_pool_location_of", C.c_int, vp)
_decl("tsb_pool_device", C.c_int, vp)
_decl("tsb_ledger_create", st, C.c_int, i64, P(vp))
_decl("tsb_ledger_destroy", None, vp)
_decl("tsb_ledger_request", st, vp, i64, i32, i64, P(C.c_int))
_decl("tsb_ledger_release", st, vp, i64, P(Grant), i64, P(i64))
for _n in ("reserved", "capacity", "deferred"):
    _decl(f"tsb_ledger_{_n}", i64, vp)
_decl("tsb_l1_create", st, C.c_int, P(KvShape), i64, i64, i64, vp, P(vp))
_decl("tsb_l1_destroy", None, vp)
_decl("tsb_l1_request", st, vp, i64, i32, i64, P(C.c_int), P(i32))
_decl("tsb_l1_release_request", st, vp, i64, P(Grant), i64, P(i64))
for _n in ("reserved", "capacity", "deferred", "free_pages", "num_pages", "page_bytes", "block_table_stride"):
    _decl(f"tsb_l1_{_n}", i64, vp)
_decl("tsb_l1_arena", vp, vp)
_decl("tsb_l1_set_layout", st, vp, C.c_int)
_decl("tsb_l1_layout", C.c_int, vp)
_decl("tsb_l1_layer_ptr", vp, vp, i64)
_decl("tsb_l1_block_table_host", vp, vp)
_decl("tsb_l1_block_table_device", vp, vp)
_decl("tsb_l1_sync_block_table", st, vp, vp)
_decl("tsb_ingest", st, vp, vp, P(IngestItem), i64, i64, i64, C.c_int, vp, P(vp))
_decl("tsb_ingest_device", st, vp, vp, vp, i64, i64, i64, C.c_int, vp, P(vp))
_decl("tsb_ingest_set_ce", st, C.c_int, i64)
_decl("tsb_l1_set_ce_group_bytes", st, vp, i64)
_decl("tsb_l1_ce_group_bytes", i64, vp)
_decl("tsb_ingest_tiered", st, vp, vp, vp, P(IngestItem), i64, i64, i64, C.c_int, vp, P(vp))
_decl("tsb_ingest_ce_direct_supported", C.c_int, vp, vp)
_decl("tsb_ingest_resolve_mode", st, vp, vp, P(IngestItem), i64, C.c_int, P(C.c_int))
_decl("tsb_ingest_set_scatter", st, C.c_int, C.c_int)
class PageCopy(C.Structure):
    _fields_ = [("src_row", i32), ("src_chunk", i32), ("dst_row", i32), ("dst_chunk", i32)]


_decl("tsb_l1_copy_chunks", st, vp, P(PageCopy), i64, i64, i64, vp)
_decl("tsb_scatter_device", st, vp, vp, vp, i64, i64, i64, vp)
_decl("tsb_scatter_device_packed", st, vp, vp, vp, i64, i64, i64, vp)
_decl("tsb_ingest_set_grid", st, C.c_int, C.c_int, C.c_int)
_decl("tsb_l1_device", C.c_int, vp)
_decl("tsb_l1_shape", st, vp, P(KvShape))
_decl("tsb_stage_create", st, vp, vp, P(vp))
_decl("tsb_stage_destroy", None, vp)
_decl("tsb_stage_set_hbm_tier", st, vp, vp)
_decl("tsb_stage_set_l3", st, vp, vp, C.c_int)
PREFILL_HOOK = C.CFUNCTYPE(C.c_int, vp, i64, i32, i64, vp)
_decl("tsb_stage_set_prefill_hook", st, vp, PREFILL_HOOK, vp)
_decl("tsb_stage_compute_stream", vp, vp)
_decl("tsb_stage_set_compute_stream", st, vp, vp)
_decl("tsb_stage_run", st, vp, i64, P(Queue), P(Cluster), P(f64), vp, vp, P(StageOptions), vp, P(StageRequest),
      P(StageStats))
_decl("tsb_stage_trace", st, vp, P(TraceRow), i64, P(i64))
_decl("tsb_stage_run_online", st, vp, i64, P(Queue), P(Cluster), P(f64), vp, vp, P(StageOptions), vp,
      P(StageRequest), P(StageStats))
_decl("tsb_l1_verify_synthetic", st, vp, P(IngestItem), i64, i64, i64, u64, i64, vp, P(u64))

def last_error() -> str:
    return lib.tsb_last_error().decode()
