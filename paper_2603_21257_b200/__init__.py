"""B200-native CALVO KV-ingest path (arxiv 2603.21257) behind the reference tiersim API.

Modules:
  tiersim  -- reference-shaped API (types, cost model, scheduler, TierLedger, errors)
  ingest   -- L2 pinned chunk pool, L1 paged KV cache + block_table, L2->L1 ingest kernels
  scorer   -- batched GPU service-cost scorer + schedule order
  hasher   -- warp-parallel prefix chunk hasher
All compute goes through libtsb.so (include/tsb_capi.h); importing without it fails loudly.
"""
from . import _capi  # noqa: F401  (raises ImportError if libtsb.so is missing)
from .tiersim import *  # noqa: F401,F403

__version__ = "0.1.0"
