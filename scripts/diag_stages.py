"""Per-structure stage split of the C2 step (diagnostic, not part of the bench)."""
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
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for s in sys.argv[1:] or ["1p", "2p", "3p", "2i", "up"]:
    a, r = synth.make_queries(s, B, N, R, seed=synth.query_seed(SEED, s))
    da, dr = torch.from_numpy(a).cuda(), torch.from_numpy(r).cuda()
    for _ in range(3):
        e.submit(s, da, dr, K)
    torch.cuda.synchronize()
    for flushed in (False, True):
        e.profile(True)
        e.profile_read()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0.0
        for _ in range(10):
            if flushed:
                flush.zero_()
            ev0.record()
            e.submit(s, da, dr, K)
            ev1.record()
            torch.cuda.synchronize()
            tot += ev0.elapsed_time(ev1)
        p = e.profile_read()
        e.profile(False)
        print(f"{s:4s} flushed={flushed!s:5s} total {tot / 10 * 1e3:7.1f} us | " +
              " ".join(f"{k} {v[0] / 10 * 1e3:6.1f} us ({v[1] // 10})" for k, v in p.items()), flush=True)
