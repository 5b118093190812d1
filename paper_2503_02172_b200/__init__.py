"""B200-native batched CLQA query-embedding inference (GQE / Query2Box / BetaE).

The hot path lives in libkgq.so (hand-written sm_100a CUDA behind the C ABI of
include/kgq.h); ``kgq`` is its thin ctypes binding.  Importing fails loudly if the
library has not been built -- there is no CPU fallback.
"""
from .kgq import (Engine, KgqError, STRUCTURES, MODELS, num_anchors, num_branches,  # noqa: F401
                  num_relations, shard_range, structure_id, uses_negation, embedding_width)
