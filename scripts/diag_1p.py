"""One warm 1p submit (C2 shape) for per-kernel ncu timing (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2503_02172_b200 import Engine
N, R, d, H, B, K = 14505, 237, 400, 1600, 1024, 10
SEED = 2503_02172 + 1
t = synth.make_tables("betae", N, R, d, hidden=H, seed=SEED)
e = Engine("betae", N, R, d, hidden=H, max_batch=B, max_k=K)
e.load_tables(t)
s = sys.argv[1] if len(sys.argv) > 1 else "1p"
a, r = synth.make_queries(s, B, N, R, seed=synth.query_seed(SEED, s))
da, dr = torch.from_numpy(a).cuda(), torch.from_numpy(r).cuda()
for _ in range(4):
    e.submit(s, da, dr, K)
torch.cuda.synchronize()
if len(sys.argv) > 2 and sys.argv[2] == "time":
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        e.submit(s, da, dr, K)
    e1.record()
    torch.cuda.synchronize()
    print(f"{s}: {e0.elapsed_time(e1) * 1e3 / 20:.1f} us per submit (graph replay, warm L2), launches {e.last_launch_count()}")
