"""Stage split of the C2 step as one mixed-structure submit (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2503_02172_b200 import Engine
N, R, d, H, B, K = 14505, 237, 400, 1600, 1024, 10
SEED = 2503_02172 + 1
t = synth.make_tables("betae", N, R, d, hidden=H, seed=SEED)
e = Engine("betae", N, R, d, hidden=H, max_batch=B * 14, max_k=K)
e.load_tables(t)
groups = []
for s in synth.STRUCTURES:
    a, r = synth.make_queries(s, B, N, R, seed=synth.query_seed(SEED, s))
    groups.append((s, torch.from_numpy(a).cuda().int(), torch.from_numpy(r).cuda().int()))
for _ in range(3):
    e.submit_mixed(groups, K)
torch.cuda.synchronize()
e.profile(True)
e.profile_read()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
tot = 0.0
for _ in range(5):
    ev0.record()
    e.submit_mixed(groups, K)
    ev1.record()
    torch.cuda.synchronize()
    tot += ev0.elapsed_time(ev1)
p = e.profile_read()
print(f"mixed step {tot / 5:.3f} ms | " + " ".join(f"{k} {v[0] / 5:.3f} ms ({v[1] // 5}, {v[2] / max(v[0], 1e-9) / 1e9 * 5 / 5:.0f} TF)" for k, v in p.items()))
print("launches", e.last_launch_count())
