"""Per-launch time and TFLOP/s of every tcgen05 GEMM in one C2 mixed step (diagnostic).

Pairs the host-side plan lines (KGQ_PLAN_LOG=1: M, N, K, BN, split plan, in launch order) with the
in-kernel launch spans (kgq_ktime_log) of the timed replays.  Runs with KGQ_NO_SPLIT_MLP=1 so all
GEMMs are on one stream and span start order == launch order (the headline runs the >= 8K-row MLPs
as two halves on two streams; the per-launch shapes are otherwise the same).
"""
import os
import re
import sys
import tempfile

os.environ["KGQ_PLAN_LOG"] = "1"
os.environ.setdefault("KGQ_NO_SPLIT_MLP", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2503_02172_b200 import Engine  # noqa: E402

N, R, d, H, B, K = 14505, 237, 400, 1600, 1024, 10
SEED = 2503_02172 + 1
STEPS = 5
t = synth.make_tables("betae", N, R, d, hidden=H, seed=SEED)
e = Engine("betae", N, R, d, hidden=H, max_batch=B * 14, max_k=K)
e.load_tables(t)
groups = []
for s in synth.STRUCTURES:
    a, r = synth.make_queries(s, B, N, R, seed=synth.query_seed(SEED, s))
    groups.append((s, torch.from_numpy(a).cuda().int(), torch.from_numpy(r).cuda().int()))

log = tempfile.NamedTemporaryFile(delete=False)
saved = os.dup(2)
os.dup2(log.fileno(), 2)
try:
    e.ktime(True)
    for _ in range(3):
        e.submit_mixed(groups, K)
    torch.cuda.synchronize()
    e.ktime_log()
    e.ktime_read()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(STEPS):
        e.submit_mixed(groups, K)
    ev1.record()
    torch.cuda.synchronize()
    spans = e.ktime_log()
finally:
    os.dup2(saved, 2)
plans = [ln for ln in open(log.name).read().splitlines() if ln.startswith("KGQ_PLAN")]
os.unlink(log.name)
per = len(spans) // STEPS
spans = spans[np.argsort(spans[:, 0], kind="stable")]
dur = (spans[:, 1].astype(np.float64) - spans[:, 0].astype(np.float64)).reshape(STEPS, per) / 1e3  # us
plans = plans[-per:]
step_ms = ev0.elapsed_time(ev1) / STEPS
print(f"# C2 mixed step {step_ms:.3f} ms (KGQ_NO_SPLIT_MLP={os.environ['KGQ_NO_SPLIT_MLP']}), {per} GEMM launches")
print(f"{'us':>8} {'TF/s':>6}  plan")
tot_us = tot_f = 0.0
for i, p in enumerate(plans):
    kv = dict(re.findall(r"(\w+)=(-?\d+)", p))
    m, n, k = int(kv["M"]), int(kv["N"]), int(kv["K"])
    us = float(np.median(dur[:, i]))
    fl = 2.0 * m * n * k
    tot_us += us
    tot_f += fl
    print(f"{us:8.1f} {fl / us / 1e6:6.1f}  {p[9:]}")
print(f"# sum {tot_us:.1f} us, {tot_f / 1e9:.1f} GFLOP, {tot_f / tot_us / 1e6:.1f} TFLOP/s")
