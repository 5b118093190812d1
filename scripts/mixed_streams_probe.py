"""Experiment (not a test): the C2 step (14 x 1024 BetaE queries) as kgq_submit_mixed calls over
S concurrent streams (one context each).  mode "rows": every stream runs all 14 types with its
slice of each type's 1024 rows; mode "types": the 14 types are dealt over the streams, each
stream one mixed submit of its types at 1024 rows.  Device time of the whole step, L2 flushed
between steps; the stage split of one mixed submit with profiling on is printed at the end.
usage: python scripts/mixed_streams_probe.py [rows:S | types:S ...]"""
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
ST = synth.STRUCTURES
t = synth.make_tables("betae", N, R, D, hidden=H, seed=SEED)
q = {s: synth.make_queries(s, B, N, R, seed=synth.query_seed(SEED, s)) for s in ST}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
main = torch.cuda.current_stream()


def lanes(mode, S):
    """per stream: (structures, batches, packed anchors, packed rels)"""
    out = []
    for j in range(S):
        if mode == "rows":
            lo, hi = j * B // S, (j + 1) * B // S
            ss = list(ST)
            parts = [(q[s][0][lo:hi], q[s][1][lo:hi]) for s in ss]
        else:
            ss = [s for i, s in enumerate(ST) if i % S == j]
            parts = [q[s] for s in ss]
        a = torch.cat([torch.from_numpy(p[0]).reshape(-1) for p in parts]).int().cuda()
        r = torch.cat([torch.from_numpy(p[1]).reshape(-1) for p in parts]).int().cuda()
        out.append((ss, [p[0].shape[0] for p in parts], a, r))
    return out


res = []
for arg in sys.argv[1:] or ["rows:1", "rows:2", "rows:3", "types:2"]:
    mode, S = arg.split(":")
    S = int(S)
    L = lanes(mode, S)
    engines = []
    for j in range(S):
        e = Engine("betae", N, R, D, hidden=H, max_batch=sum(L[j][1]), max_k=K)
        e.load_tables(t)
        engines.append(e)
    outs = [(torch.empty((sum(l[1]), K), device="cuda"), torch.empty((sum(l[1]), K), dtype=torch.int32, device="cuda"))
            for l in L]
    streams = [torch.cuda.Stream() for _ in range(S)]

    def step():
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for st in streams:
            st.wait_event(e0)
        for j in range(S):
            engines[j].submit_mixed_packed(L[j][0], L[j][1], L[j][2], L[j][3], K, outs[j], stream=streams[j])
        for st in streams:
            ev = torch.cuda.Event()
            ev.record(st)
            main.wait_event(ev)
        e1.record(main)
        return e0, e1

    for _ in range(4):
        step()
    torch.cuda.synchronize()
    for e in engines:
        e.check_errors()
    ms = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = step()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    ms.sort()
    r = {"mode": mode, "streams": S, "ms_median": ms[len(ms) // 2], "ms_min": ms[0],
         "qps": 14 * B / (ms[len(ms) // 2] / 1e3)}
    print(json.dumps(r), flush=True)
    res.append(r)
    if S == 1:  # stage split of the one-stream mixed submit
        e = engines[0]
        e.profile(True)
        e.profile_read()
        for _ in range(5):
            step()
        torch.cuda.synchronize()
        p = e.profile_read()
        e.profile(False)
        print(json.dumps({"stages_ms": {k: v[0] / 5 for k, v in p.items()},
                          "tflops": {k: v[2] / max(v[0], 1e-9) / 1e9 for k, v in p.items()}}), flush=True)
    for e in engines:
        e.close()
