"""Float64 CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product path never does.  See kgq_oracle.py.
"""
from .kgq_oracle import *  # noqa: F401,F403
from .kgq_oracle import Model, PLANS, STRUCTURES, topk, merge_topk, shard_range  # noqa: F401
