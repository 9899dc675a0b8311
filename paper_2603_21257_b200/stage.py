"""Load stage: the real-time L2->L1 dispatcher (tsb_stage_*), SimEngine's dispatch semantics with
real bytes (engine.cpp:290-302, 341-355, 405-446, 258-282)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _capi as capi
from ._capi import lib
from .ingest import AUTO, ChunkPool, PagedKVCache
from .tiersim import ClusterConfig, CostModelPair, PolicyKind, QueueArrays, check, cost_models_from_config

TRACE_KINDS = {0: "arrival", 1: "transfer_done", 2: "allocation_grant", 3: "compute_done", 4: "dispatch_wake"}


@dataclass
class StageResult:
    requests: np.ndarray  # structured: request_id, pick_position, deferred_chunks, chunks, bytes, *_ms
    stats: dict
    trace: Optional[np.ndarray] = None


class LoadStage:
    def __init__(self, l1: PagedKVCache, pool: ChunkPool):
        h = C.c_void_p()
        check(lib.tsb_stage_create(l1.handle, pool.handle, C.byref(h)))
        self._h = h
        self.l1, self.pool = l1, pool

    def set_hbm_tier(self, hbm_pool: Optional[ChunkPool]):
        """Chunks whose slot is < 0 in run()/run_online() come from slot ~slot of hbm_pool (this GPU's
        or a peer's HBM) instead of crossing the host link; None clears the tier."""
        check(lib.tsb_stage_set_hbm_tier(self._h, hbm_pool.handle if hbm_pool is not None else None))
        self.hbm_pool = hbm_pool

    def set_l3(self, l3_pool: Optional[ChunkPool], copy_threads: int = 4):
        """Online mode: blocks start in `l3_pool` (slots name L3 chunks) and make the network hop
        L3 -> L2 for real into slots of this stage's pool, granted by a TierLedger(L2) + slot free
        list and released after the L2 -> L1 hop (engine.cpp:341-364, 405-425, 264).  None detaches."""
        check(lib.tsb_stage_set_l3(self._h, l3_pool.handle if l3_pool is not None else None, int(copy_threads)))
        self.l3_pool = l3_pool

    def set_prefill_hook(self, fn):
        """fn(q_index, bt_row, layer, stream_ptr) -> None enqueues layer `layer` of request q_index's
        prefill on the stage's compute stream (after the stage made that stream wait for the layer's
        fence).  It replaces the K6 timer; None restores it.  An exception fails the stage call."""
        if fn is None:
            self._hook = None
            check(lib.tsb_stage_set_prefill_hook(self._h, capi.PREFILL_HOOK(), None))
            return

        def tramp(_user, q_index, bt_row, layer, stream):
            try:
                fn(int(q_index), int(bt_row), int(layer), int(stream or 0))
                return 0
            except Exception as e:  # noqa: BLE001 -- reported through the stage status
                self.hook_error = e
                return 1

        self.hook_error = None
        self._hook = capi.PREFILL_HOOK(tramp)  # kept alive with the stage
        # Prefill runs on a torch-owned lowest-priority stream: torch tensors the consumer touches
        # there (pinned staging included) may outlive the stage without referencing a dead stream.
        if getattr(self, "_compute", None) is None:
            self._compute = torch.cuda.Stream(device=torch.device("cuda", self.l1.device), priority=0)
            check(lib.tsb_stage_set_compute_stream(self._h, self._compute.cuda_stream))
        check(lib.tsb_stage_set_prefill_hook(self._h, self._hook, None))

    @property
    def compute_stream(self):
        if getattr(self, "_compute", None) is not None:
            return self._compute
        return torch.cuda.ExternalStream(lib.tsb_stage_compute_stream(self._h), device=torch.device("cuda", self.l1.device))

    def close(self):
        if getattr(self, "_h", None) and lib is not None:  # lib is None during interpreter exit
            lib.tsb_stage_destroy(self._h)
            self._h = None
        # drop the tiers so a closed stage does not keep an L1 arena or a pool alive
        self.l1 = self.pool = self.hbm_pool = self.l3_pool = None

    __del__ = close

    def run_online(self, queue: QueueArrays, slot_lists: Sequence[Sequence[int]], config: ClusterConfig,
                   models: Optional[CostModelPair] = None, policy: int = PolicyKind.Fifo, mode: int = AUTO,
                   prefill_ctas: int = 0, verify_seed: int = 0, stream=None, pace_network: bool = False,
                   record_trace: bool = False, reuse_l1: bool = False) -> StageResult:
        """Real-time replay: arrivals at their arrival_time, SimEngine's control loop under
        config.control_mode / allocation_mode (tsb_stage_run_online).  requests['done_ms'] -
        requests['arrival_ms'] is each TTFT.  verify_seed (opt-in, perturbs timing): check every page
        of each request before release.  pace_network: with an L3 store, each network hop lasts at
        least transfer_base_latency + bytes / network_bandwidth.  reuse_l1: a chunk already resident
        in a live request's pages is replicated HBM -> HBM instead of crossing the link (no L3)."""
        return self.run(queue, slot_lists, config, models, policy, mode, prefill=True, prefill_ctas=prefill_ctas,
                        verify_seed=verify_seed, stream=stream, record_trace=record_trace,
                        pace_network=pace_network, reuse_l1=reuse_l1, _fn=lib.tsb_stage_run_online)

    def run(self, queue: QueueArrays, slot_lists: Sequence[Sequence[int]], config: ClusterConfig,
            models: Optional[CostModelPair] = None, policy: int = PolicyKind.Fifo, mode: int = AUTO,
            layer_events: bool = False, prefill: bool = False, prefill_ctas: int = 0, record_trace: bool = False,
            verify_seed: int = 0, stream=None, pace_network: bool = False, reuse_l1: bool = False,
            _fn=None) -> StageResult:
        fn = _fn or lib.tsb_stage_run
        models = models or cost_models_from_config(config)
        offs = np.zeros(len(slot_lists) + 1, np.int64)
        np.cumsum([len(s) for s in slot_lists], out=offs[1:])
        slots = np.concatenate([np.asarray(s, np.int64) for s in slot_lists]) if len(slot_lists) else np.zeros(0, np.int64)
        slots = np.ascontiguousarray(slots, np.int64)
        opt = capi.StageOptions(int(mode), int(policy), int(layer_events), int(prefill), int(prefill_ctas),
                                int(record_trace), int(verify_seed), int(pace_network), int(reuse_l1))
        res = (capi.StageRequest * max(queue.n, 1))()
        stats = capi.StageStats()
        qs = queue.struct()
        s = (stream or torch.cuda.current_stream()).cuda_stream
        rc = fn(self._h, queue.n, C.byref(qs), C.byref(config.struct()), models.array(),
                offs.ctypes.data, slots.ctypes.data, C.byref(opt), s, res, C.byref(stats))
        if rc != capi.TSB_OK and getattr(self, "hook_error", None) is not None:
            err, self.hook_error = self.hook_error, None
            raise err
        check(rc)
        dt = np.dtype([(n, np.int64 if t in (capi.i64,) else np.int32 if t is capi.i32 else np.float64)
                       for n, t in capi.StageRequest._fields_])
        arr = np.frombuffer(bytes(res), dtype=dt, count=queue.n) if queue.n else np.zeros(0, dt)
        st = {n: getattr(stats, n) for n, _ in capi.StageStats._fields_}
        trace = None
        if record_trace:
            n = C.c_int64()
            check(lib.tsb_stage_trace(self._h, None, 0, C.byref(n)))
            rows = (capi.TraceRow * max(n.value, 1))()
            check(lib.tsb_stage_trace(self._h, rows, n.value, C.byref(n)))
            tdt = np.dtype([(f, np.float64 if t is capi.f64 else np.uint64 if t is capi.u64 else
                             np.int64 if t is capi.i64 else np.int32) for f, t in capi.TraceRow._fields_])
            trace = np.frombuffer(bytes(rows), dtype=tdt, count=n.value)
        return StageResult(arr, st, trace)
