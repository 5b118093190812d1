"""Experiment (not a test): the C2 step (14 x 1024 BetaE queries, one per-type kgq_submit each)
with the 14 submits spread round-robin over S streams (one context per stream), vs S = 1.
Device time of the whole step (event on a start stream, every stream joins an end event), L2
flushed between steps.  usage: python scripts/multistream_probe.py [S ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2503_02172_b200 import Engine  # noqa: E402

N, R, D, H, B, K = 14505, 237, 400, 1600, 1024, 10
SEED = 2503_02172 + 1
t = synth.make_tables("betae", N, R, D, hidden=H, seed=SEED)
qs = {}
for s in synth.STRUCTURES:
    a, r = synth.make_queries(s, B, N, R, seed=synth.query_seed(SEED, s))
    qs[s] = (torch.from_numpy(a).cuda(), torch.from_numpy(r).cuda())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {}
engines = []
for S in [int(x) for x in (sys.argv[1:] or ["1", "2", "3", "4"])]:
    while len(engines) < S:
        e = Engine("betae", N, R, D, hidden=H, max_batch=B, max_k=K)
        e.load_tables(t)
        engines.append(e)
    streams = [torch.cuda.Stream() for _ in range(S)]
    outs = {s: (torch.empty((B, K), device="cuda"), torch.empty((B, K), dtype=torch.int32, device="cuda"))
            for s in synth.STRUCTURES}
    main = torch.cuda.current_stream()

    def step():
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for st in streams:
            st.wait_event(e0)
        for i, s in enumerate(synth.STRUCTURES):
            j = i % S
            engines[j].submit(s, *qs[s], K, out=outs[s], stream=streams[j])
        for st in streams:
            ev = torch.cuda.Event()
            ev.record(st)
            main.wait_event(ev)
        e1.record(main)
        return e0, e1

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ms = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = step()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    ms.sort()
    out[S] = {"ms_median": ms[len(ms) // 2], "ms_min": ms[0], "qps": 14 * B / (ms[len(ms) // 2] / 1e3)}
    print(json.dumps({"streams": S, **out[S], "pdl": os.environ.get("KGQ_PDL", "default")}), flush=True)
