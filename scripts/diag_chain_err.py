"""Full-size chain-embedding error vs the oracle per structure (diagnostic, not a test)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import oracle as O
import synth
from paper_2503_02172_b200 import Engine
N, R, d, H, B = 14505, 237, 400, 1600, 1024
seed = 2503_02172 + 1
t = synth.make_tables("betae", N, R, d, hidden=H, seed=seed)
e = Engine("betae", N, R, d, hidden=H, max_batch=B, max_k=16)
e.load_tables(t)
m = O.Model("betae", t, dim=d)
rng = np.random.default_rng(0)
out = []
for s in synth.ALL_STRUCTURES:
    a, r = synth.make_queries(s, B, N, R, seed=synth.query_seed(seed, s))
    rows = np.unique(np.r_[rng.integers(0, B, size=1), B - 1])
    qe = e.query_embedding(s, torch.from_numpy(a).cuda(), torch.from_numpy(r).cuda()).cpu().numpy()[rows].astype(np.float64)
    ref = m.query_embedding(s, a[rows], r[rows])
    floor = 1e-2 * np.max(np.abs(ref), axis=-1, keepdims=True)
    err = np.abs(qe - ref) / np.maximum(np.abs(ref), floor)
    out.append(f"{s}:{err.max():.3g}")
print(" ".join(out))
