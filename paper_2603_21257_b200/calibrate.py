"""Closing the loop from measured ingest to scheduler cost.

The reference scores requests with a linear loading model T_load(cached tokens) = ls * n + li
(cost_model.cpp:52-71) whose default comes from assumed bandwidths (cost_models_from_config,
cost_model.cpp:73-85) -- or from measured samples fitted by fit_linear (cost_model.cpp:14-50) after
read_samples_csv (cost_model.cpp:105-123).  Here the samples are the real L2 -> L1 hops: every
stage run reports, per request, its cached tokens and the CUDA-event span of its ingest
(ingest_begin_ms -> resident_ms), and, for prefill without layer pipelining, its compute tokens
and prefill span (resident_ms -> done_ms).  They are written in read_samples_csv format, read
back through the reference-shaped reader, fitted, and the fitted CostModelPair goes to the GPU
scorer (K4) like any other model.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .tiersim import (ClusterConfig, CostModelPair, LinearCostModel, LinearFit, TokenSample, cost_models_from_config,
                      fit_linear, read_samples_csv, write_samples_csv)


def ingest_samples(requests: np.ndarray) -> list[TokenSample]:
    """(cached tokens, seconds of the request's L2 -> L1 hops) per request that moved chunks.
    Requests with a deferred chunk reservation are left out: their span from first hop to
    residency includes the wait for pages that a release granted later, which the reference
    models as TierLedger deferral (engine.cpp:38-49), not as transfer time (engine.cpp:206-207)."""
    out = []
    for r in requests:
        if r["chunks"] > 0 and r["deferred_chunks"] == 0:
            out.append(TokenSample(int(r["cached_tokens"]), float(r["resident_ms"] - r["ingest_begin_ms"]) * 1e-3))
    return out


def compute_samples(requests: np.ndarray) -> list[TokenSample]:
    """(compute tokens, prefill seconds) per request, for runs whose prefill starts once the request
    is resident (layer_events off).  Prefills run one at a time in pick order on the compute
    stream, so a request's prefill starts at max(its residency, the previous prefill's end)."""
    out, prev_done = [], 0.0
    for r in requests[np.argsort(requests["pick_position"], kind="stable")]:
        start = max(float(r["resident_ms"]), prev_done)
        out.append(TokenSample(int(r["compute_tokens"]), (float(r["done_ms"]) - start) * 1e-3))
        prev_done = float(r["done_ms"])
    return out


@dataclass
class Calibration:
    load: LinearFit
    comp: Optional[LinearFit]
    models: CostModelPair
    default: CostModelPair
    load_csv: str
    comp_csv: Optional[str]


def calibrate(results, config: ClusterConfig, out_dir: str, fit_compute: bool = False) -> Calibration:
    """Fit T_load (and optionally T_comp) from one or more StageResults; the CSVs are the audit
    trail in the reference's sample format."""
    os.makedirs(out_dir, exist_ok=True)
    results = results if isinstance(results, (list, tuple)) else [results]
    load_csv = os.path.join(out_dir, "t_load_samples.csv")
    write_samples_csv(load_csv, [s for r in results for s in ingest_samples(r.requests)])
    load = fit_linear((s.tokens, s.seconds) for s in read_samples_csv(load_csv))
    default = cost_models_from_config(config)
    comp, comp_csv = None, None
    comp_model = default.comp
    if fit_compute:
        comp_csv = os.path.join(out_dir, "t_comp_samples.csv")
        write_samples_csv(comp_csv, [s for r in results for s in compute_samples(r.requests)])
        comp = fit_linear((s.tokens, s.seconds) for s in read_samples_csv(comp_csv))
        comp_model = comp.model
    return Calibration(load, comp, CostModelPair(LinearCostModel(load.model.slope, load.model.intercept), comp_model),
                       default, load_csv, comp_csv)
