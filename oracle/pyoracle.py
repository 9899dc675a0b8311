"""ctypes loader for the oracle libraries -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg import
this module, and only as the checker or the CPU arm.  The product package never does.

  restate() -> oracle/build/libtsb_oracle.so   (C restatement, tsb_oracle.c; built anywhere)
  ref()     -> oracle/_ref/libtiersim_ref.so    (the reference's own sources + ref_adapter.cpp;
                                                 None when it was not built here)
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
RESTATE_SO = HERE / "build" / "libtsb_oracle.so"
REF_SO = HERE / "_ref" / "libtiersim_ref.so"
ACCEPTANCE = HERE / "_ref" / "acceptance_test"

vp, i64, i32, u64, f64 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.c_double


class OrcCluster(C.Structure):
    _fields_ = [
        ("network_bandwidth", f64), ("pcie_bandwidth", f64), ("transfer_base_latency", f64),
        ("l1_capacity", i64), ("l2_capacity", i64), ("bytes_per_token", i64), ("block_size_tokens", i64),
        ("compute_base", f64), ("compute_per_token", f64), ("compute_quadratic", f64),
        ("allocation_mode", i32), ("control_mode", i32),
    ]


class OrcQueue(C.Structure):
    _fields_ = [(n, vp) for n in ("id", "arrival", "context_tokens", "query_tokens", "cache_hit_ratio", "flags",
                                  "deadline", "measured_t_load", "measured_t_comp")]


class OrcShape(C.Structure):
    _fields_ = [(n, i64) for n in ("layers", "kv_heads", "head_dim", "dtype_bytes", "chunk_tokens", "page_tokens",
                                   "tp_size", "tp_rank")]


class OrcItem(C.Structure):
    _fields_ = [("src_slot", i64), ("bt_row", i32), ("chunk_index", i32)]


def cluster_struct(cfg) -> OrcCluster:
    c = OrcCluster()
    for name, _ in OrcCluster._fields_:
        v = getattr(cfg, name)
        setattr(c, name, int(v) if name.endswith("mode") else v)
    return c


def queue_struct(q) -> OrcQueue:
    """q: paper_2603_21257_b200.tiersim.QueueArrays-like (numpy attributes)."""
    s = OrcQueue()
    for name, _ in OrcQueue._fields_:
        setattr(s, name, getattr(q, name).ctypes.data)
    return s


def _build(target: str) -> None:
    subprocess.run(["make", "-s", "-C", str(HERE), target], check=True)


_restate = None
_ref = None


def restate():
    global _restate
    if _restate is None:
        if not RESTATE_SO.exists():
            _build("restate")
        lib = C.CDLL(str(RESTATE_SO))
        d = _declare
        d(lib, "orc_kv_bytes_per_token", C.c_int, i64, i64, i64, i64, C.POINTER(i64))
        d(lib, "orc_cached_token_count", i64, i64, f64, i64)
        d(lib, "orc_compute_token_count", i64, i64, i64, f64, i64)
        d(lib, "orc_predict", f64, f64, f64, i64)
        d(lib, "orc_cost_models_from_config", None, C.POINTER(OrcCluster), C.POINTER(f64))
        d(lib, "orc_fit_linear", C.c_int, i64, vp, vp, C.POINTER(f64), C.POINTER(f64), C.POINTER(C.c_int),
          C.POINTER(C.c_int))
        d(lib, "orc_score_queue", C.c_int, i64, C.POINTER(OrcQueue), C.c_int, C.POINTER(f64), C.POINTER(OrcCluster),
          vp, vp, vp, C.POINTER(i64))
        d(lib, "orc_sort_order", C.c_int, i64, vp, vp, vp, vp)
        d(lib, "orc_drain_order", C.c_int, i64, vp, vp, vp, vp)
        d(lib, "orc_ledger_new", vp, i64)
        d(lib, "orc_ledger_free", None, vp)
        d(lib, "orc_ledger_request", C.c_int, vp, i64, i32, i64, C.POINTER(C.c_int))
        d(lib, "orc_ledger_release", C.c_int, vp, i64, vp, vp, vp, i64, C.POINTER(i64))
        d(lib, "orc_ledger_reserved", i64, vp)
        d(lib, "orc_ledger_deferred", i64, vp)
        d(lib, "orc_pages_new", vp, i64)
        d(lib, "orc_pages_free", None, vp)
        d(lib, "orc_pages_take", i64, vp, i64, vp)
        d(lib, "orc_pages_give", None, vp, i64, vp)
        d(lib, "orc_pages_available", i64, vp)
        d(lib, "orc_scatter_ref", None, C.POINTER(OrcShape), vp, i64, vp, vp, i64, i64, vp, i64, i64, C.c_int)
        d(lib, "orc_scatter_ref_layout", None, C.POINTER(OrcShape), vp, i64, vp, vp, i64, i64, vp, i64, i64, C.c_int,
          C.c_int)
        d(lib, "orc_scatter_ref_window", None, C.POINTER(OrcShape), vp, i64, vp, vp, i64, i64, vp, i64, i64, C.c_int,
          C.c_int)
        d(lib, "orc_mix64", u64, u64)
        d(lib, "orc_synth_word", u64, u64, u64)
        d(lib, "orc_synth_fill", None, u64, u64, u64, vp, C.c_int)
        d(lib, "orc_token_id", C.c_uint32, u64, u64, u64)
        d(lib, "orc_gen_tokens", None, u64, i64, vp, vp, vp, vp, C.c_int)
        d(lib, "orc_fnv1a_bytes", u64, u64, vp, C.c_size_t)
        d(lib, "orc_chunk_digest", u64, vp)
        d(lib, "orc_chain", u64, u64, u64)
        d(lib, "orc_hash_prefix_chunks", i64, i64, vp, vp, vp, vp, C.c_int)
        _restate = lib
    return _restate


def ref():
    """The compiled reference (None if /root/reference was not available to build it)."""
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            if Path("/root/reference/proj/core/src").is_dir():
                _build("ref")
            else:
                return None
        lib = C.CDLL(str(REF_SO))
        d = _declare
        d(lib, "ref_last_error", C.c_char_p)
        d(lib, "ref_kv_bytes_per_token", C.c_int, i64, i64, i64, i64, C.POINTER(i64))
        d(lib, "ref_block_plan", C.c_int, C.POINTER(OrcQueue), i64, C.POINTER(OrcCluster), *([C.POINTER(i64)] * 5))
        d(lib, "ref_cost_models_from_config", None, C.POINTER(OrcCluster), C.POINTER(f64))
        d(lib, "ref_fit_linear", C.c_int, i64, vp, vp, C.POINTER(f64))
        d(lib, "ref_score_queue", C.c_int, i64, C.POINTER(OrcQueue), C.c_int, C.POINTER(f64), C.POINTER(OrcCluster),
          vp, vp, vp, C.POINTER(i64))
        d(lib, "ref_sort_order", C.c_int, i64, C.POINTER(OrcQueue), C.c_int, C.POINTER(f64), C.POINTER(OrcCluster), vp)
        d(lib, "ref_drain_order", C.c_int, i64, C.POINTER(OrcQueue), C.c_int, C.POINTER(f64), C.POINTER(OrcCluster), vp)
        d(lib, "ref_ledger_new", vp, C.c_int, i64)
        d(lib, "ref_ledger_free", None, vp)
        d(lib, "ref_ledger_request", C.c_int, vp, i64, i32, i64, C.POINTER(C.c_int))
        d(lib, "ref_ledger_release", C.c_int, vp, i64, vp, vp, vp, i64, C.POINTER(i64))
        d(lib, "ref_ledger_reserved", i64, vp)
        d(lib, "ref_ledger_deferred", i64, vp)
        d(lib, "ref_config_fingerprint", u64, C.POINTER(OrcCluster), C.c_int, u64)
        d(lib, "ref_generate_workload", i64, C.c_char_p, f64, f64, f64, f64, i64, f64, u64, C.c_int, f64, vp, i64,
          i64, vp, vp, vp, vp, vp)
        d(lib, "ref_assign_slos", C.c_int, i64, C.POINTER(OrcQueue), C.POINTER(OrcCluster), C.POINTER(f64), vp, i64,
          u64, vp)
        d(lib, "ref_run_simulation", C.c_int, i64, C.POINTER(OrcQueue), C.POINTER(OrcCluster), C.c_int,
          C.POINTER(f64), u64, vp, C.POINTER(f64))
        _ref = lib
    return _ref


def _declare(lib, name, restype, *argtypes):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)


# ---- convenience wrappers used by tests and bench ---------------------------------------------
def score_queue(q, policy: int, models, cfg, which: str = "restate"):
    """Returns (status, err_index, t_load, t_comp, primary) from the restatement or the reference."""
    n = q.n
    tl, tc, pr = (np.zeros(n, np.float64) for _ in range(3))
    err = i64(-1)
    m = (f64 * 4)(*models)
    qs, cs = queue_struct(q), cluster_struct(cfg)
    if which == "ref":
        st = ref().ref_score_queue(n, C.byref(qs), policy, m, C.byref(cs), tl.ctypes.data, tc.ctypes.data,
                                   pr.ctypes.data, C.byref(err))
    else:
        st = restate().orc_score_queue(n, C.byref(qs), policy, m, C.byref(cs), tl.ctypes.data, tc.ctypes.data,
                                       pr.ctypes.data, C.byref(err))
    return st, err.value, tl, tc, pr


def sort_order(primary, arrival, ids) -> np.ndarray:
    p = np.ascontiguousarray(primary, np.float64)
    a = np.ascontiguousarray(arrival, np.float64)
    i = np.ascontiguousarray(ids, np.int64)
    out = np.empty(len(p), np.int64)
    restate().orc_sort_order(len(p), p.ctypes.data, a.ctypes.data, i.ctypes.data, out.ctypes.data)
    return out


def ref_sort_order(q, policy, models, cfg) -> np.ndarray:
    out = np.empty(q.n, np.int64)
    m = (f64 * 4)(*models)
    qs, cs = queue_struct(q), cluster_struct(cfg)
    st = ref().ref_sort_order(q.n, C.byref(qs), policy, m, C.byref(cs), out.ctypes.data)
    assert st == 0, ref().ref_last_error()
    return out


def ref_drain_order(q, policy, models, cfg) -> np.ndarray:
    out = np.empty(q.n, np.int64)
    m = (f64 * 4)(*models)
    qs, cs = queue_struct(q), cluster_struct(cfg)
    st = ref().ref_drain_order(q.n, C.byref(qs), policy, m, C.byref(cs), out.ctypes.data)
    assert st == 0, ref().ref_last_error()
    return out


def scatter_ref(shape, pool: np.ndarray, items: np.ndarray, block_table: np.ndarray, num_pages: int,
                layer_lo: int = 0, layer_hi=None, threads: int = 1, arena: np.ndarray = None,
                layout: int = 0) -> np.ndarray:
    """items: structured array (src_slot i64, bt_row i32, chunk_index i32).  layout: 0 flash-attn,
    1 FlashInfer NHD, 2 FlashInfer HND (orc_scatter_ref_layout)."""
    layer_hi = shape.layers if layer_hi is None else layer_hi
    hl = shape.kv_heads // shape.tp_size
    layer_bytes = 2 * num_pages * shape.page_tokens * hl * shape.head_dim * shape.dtype_bytes
    if arena is None:
        arena = np.zeros(shape.layers * layer_bytes, dtype=np.uint8)
    s = OrcShape(shape.layers, shape.kv_heads, shape.head_dim, shape.dtype_bytes, shape.chunk_tokens,
                 shape.page_tokens, shape.tp_size, shape.tp_rank)
    bt = np.ascontiguousarray(block_table, np.int32)
    restate().orc_scatter_ref_layout(C.byref(s), pool.ctypes.data, len(items), items.ctypes.data, bt.ctypes.data,
                                     bt.shape[1], num_pages, arena.ctypes.data, layer_lo, layer_hi, threads, layout)
    return arena


def scatter_ref_window(shape, pool: np.ndarray, items: np.ndarray, block_table: np.ndarray, num_pages: int,
                       layer_lo: int, layer_hi: int, threads: int = 1, layout: int = 0) -> np.ndarray:
    """scatter_ref of layers [layer_lo, layer_hi) only; returns just those layers of the arena."""
    hl = shape.kv_heads // shape.tp_size
    layer_bytes = 2 * num_pages * shape.page_tokens * hl * shape.head_dim * shape.dtype_bytes
    arena = np.zeros((layer_hi - layer_lo) * layer_bytes, dtype=np.uint8)
    s = OrcShape(shape.layers, shape.kv_heads, shape.head_dim, shape.dtype_bytes, shape.chunk_tokens,
                 shape.page_tokens, shape.tp_size, shape.tp_rank)
    bt = np.ascontiguousarray(block_table, np.int32)
    restate().orc_scatter_ref_window(C.byref(s), pool.ctypes.data, len(items), items.ctypes.data, bt.ctypes.data,
                                     bt.shape[1], num_pages, arena.ctypes.data, layer_lo, layer_hi, threads, layout)
    return arena


def synth_fill(seed: int, first_word: int, n_words: int, threads: int = 1) -> np.ndarray:
    out = np.empty(n_words, np.uint64)
    restate().orc_synth_fill(seed, first_word, n_words, out.ctypes.data, threads)
    return out


def gen_tokens(seed, offsets, doc, shared_len, threads: int = 1) -> np.ndarray:
    offsets = np.ascontiguousarray(offsets, np.int64)
    doc = np.ascontiguousarray(doc, np.int64)
    sl = np.ascontiguousarray(shared_len, np.int64)
    out = np.empty(int(offsets[-1]), np.int32)
    restate().orc_gen_tokens(seed, len(offsets) - 1, offsets.ctypes.data, doc.ctypes.data, sl.ctypes.data,
                             out.ctypes.data, threads)
    return out


def hash_prefix_chunks(offsets, tokens, threads: int = 1) -> np.ndarray:
    offsets = np.ascontiguousarray(offsets, np.int64)
    tokens = np.ascontiguousarray(tokens, np.int32)
    lens = np.diff(offsets)
    coff = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens // 256, out=coff[1:])
    out = np.empty(max(int(coff[-1]), 1), np.uint64)
    n = restate().orc_hash_prefix_chunks(len(lens), offsets.ctypes.data, tokens.ctypes.data, coff.ctypes.data,
                                         out.ctypes.data, threads)
    return out[:n]


def generate_workload(profile: str, count: int, seed: int, qps: float = 1.0, hit_fixed: float = 1.0,
                      hit_choices=None, ctx_mean=0.0, ctx_cv=0.5, q_mean=0.0, q_cv=0.5):
    """generate_workload (workload.cpp:70-99) through the compiled reference."""
    r = ref()
    if r is None:
        raise RuntimeError("compiled reference not available")
    ids, ctx, qry = (np.empty(count, np.int64) for _ in range(3))
    arr, hit = (np.empty(count, np.float64) for _ in range(2))
    ch = np.ascontiguousarray(hit_choices if hit_choices is not None else [], np.float64)
    n = r.ref_generate_workload(profile.encode(), ctx_mean, ctx_cv, q_mean, q_cv, count, qps, seed,
                                1 if hit_choices is not None else 0, hit_fixed, ch.ctypes.data, len(ch), count,
                                ids.ctypes.data, arr.ctypes.data, ctx.ctypes.data, qry.ctypes.data, hit.ctypes.data)
    assert n == count, r.ref_last_error()
    return ids, arr, ctx, qry, hit
