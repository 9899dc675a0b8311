"""Batched service-cost scorer + schedule order on the GPU (K4 + K5 via tsb_score_queue*).

Replaces the per-request estimate_service_cost / priority_key calls and the O(N^2) pick_next drain
(cost_model.cpp:56-71, scheduler.cpp:39-100) for a whole queue at once.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np
import torch

from . import _capi as capi
from ._capi import lib
from .tiersim import ClusterConfig, CostModelPair, QueueArrays, RequestSpec, check, cost_models_from_config


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class DeviceQueue:
    """A RequestSpec queue resident in HBM (torch tensors), viewed as tsb_queue."""

    def __init__(self, q: QueueArrays, device: int = 0):
        dev = torch.device("cuda", device)
        self.n = q.n
        self.tensors = {name: torch.from_numpy(np.ascontiguousarray(getattr(q, name))).to(dev)
                        for name, _ in QueueArrays.FIELDS}

    def struct(self) -> capi.Queue:
        s = capi.Queue()
        for name, _ in QueueArrays.FIELDS:
            setattr(s, name, self.tensors[name].data_ptr())
        return s


class BatchScorer:
    def __init__(self, device: int = 0, capacity: int = 1 << 17):
        if not torch.cuda.is_available():
            raise RuntimeError("BatchScorer needs a CUDA device (no CPU fallback)")
        self.device = device
        h = C.c_void_p()
        check(lib.tsb_scorer_create(device, capacity, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:  # lib is None during interpreter exit
            lib.tsb_scorer_destroy(self._h)
            self._h = None

    # -- host arrays in, host arrays out (the drop-in form) -----------------------------------
    def score(self, q: QueueArrays, policy: int, models: CostModelPair, config: ClusterConfig,
              stream=None):
        n = q.n
        t_load = np.empty(n, np.float64)
        t_comp = np.empty(n, np.float64)
        primary = np.empty(n, np.float64)
        order = np.empty(n, np.int64)
        qs = q.struct()
        check(lib.tsb_score_queue(self._h, _stream_ptr(stream), n, C.byref(qs), int(policy), models.array(),
                                  C.byref(config.struct()), t_load.ctypes.data, t_comp.ctypes.data,
                                  primary.ctypes.data, order.ctypes.data))
        return t_load, t_comp, primary, order

    # -- device-resident queue (the hot path) ------------------------------------------------
    def score_device(self, dq: DeviceQueue, policy: int, models: CostModelPair, config: ClusterConfig,
                     out: Optional[dict] = None, check_errors: bool = True, stream=None) -> dict:
        n = dq.n
        dev = torch.device("cuda", self.device)
        if out is None:
            out = {
                "t_load": torch.empty(n, dtype=torch.float64, device=dev),
                "t_comp": torch.empty(n, dtype=torch.float64, device=dev),
                "primary": torch.empty(n, dtype=torch.float64, device=dev),
                "order": torch.empty(n, dtype=torch.int64, device=dev),
            }
        err = C.c_int64(-1)
        qs = dq.struct()
        check(lib.tsb_score_queue_device(self._h, _stream_ptr(stream), n, C.byref(qs), int(policy), models.array(),
                                         C.byref(config.struct()), out["t_load"].data_ptr(),
                                         out["t_comp"].data_ptr(), out["primary"].data_ptr(),
                                         out["order"].data_ptr(), C.byref(err) if check_errors else None))
        out["err_index"] = err.value
        return out

    def order_specs(self, specs: Sequence[RequestSpec], policy: int, costs: Optional[dict] = None,
                    models: Optional[CostModelPair] = None, config: Optional[ClusterConfig] = None):
        config = config or ClusterConfig()
        models = models or cost_models_from_config(config)
        q = QueueArrays.from_specs(specs, costs=costs)
        return self.score(q, policy, models, config)[3]
