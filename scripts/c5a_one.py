"""One C5a case (2M entities, d 400) for ncu: python scripts/c5a_one.py gqe|betae 1p|2u B [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
from paper_2503_02172_b200 import Engine  # noqa: E402
model, s, B = sys.argv[1], sys.argv[2], int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
N, R, d = 2_000_000, 200, 400
t = synth.make_tables(model, N, R, d, hidden=1600, seed=77)
e = Engine(model, N, R, d, hidden=1600, max_batch=max(B, 8), max_k=16)
e.load_tables(t)
a, r = synth.make_queries(s, B, N, R, seed=5)
da, dr = torch.from_numpy(a).cuda(), torch.from_numpy(r).cuda()
for _ in range(reps):
    e.submit(s, da, dr, 10)
torch.cuda.synchronize()
e.check_errors()
print("ok")
