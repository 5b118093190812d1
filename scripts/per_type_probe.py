"""Per-type BetaE submit q/s at the C2 shape (diagnostic; the bench's per_type form, fewer steps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2503_02172_b200 import Engine  # noqa: E402

N, R, d, H, B, K = 14505, 237, 400, 1600, 1024, 10
SEED = 2503_02172 + 1
types = sys.argv[1].split(",") if len(sys.argv) > 1 else list(synth.STRUCTURES)
t = synth.make_tables("betae", N, R, d, hidden=H, seed=SEED)
e = Engine("betae", N, R, d, hidden=H, max_batch=B, max_k=K)
e.load_tables(t)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = {}
for s in types:
    a, r = synth.make_queries(s, B, N, R, seed=synth.query_seed(SEED, s))
    a, r = torch.from_numpy(a).cuda(), torch.from_numpy(r).cuda()
    for _ in range(3):
        e.submit(s, a, r, K)
    tot = 0.0
    for _ in range(10):
        flush.zero_()
        torch.cuda.synchronize()
        ev0.record()
        e.submit(s, a, r, K)
        ev1.record()
        torch.cuda.synchronize()
        tot += ev0.elapsed_time(ev1)
    out[s] = round(B / (tot / 10 / 1e3) / 1e6, 3)
print(out)
