"""Chain-embedding and full-row distance errors vs the oracle per structure (diagnostic, not a
test).  Prints one JSON line per config: for every structure the max element-wise relative
error of the query embedding under two floors (1e-2 and 1e-3 of the row max) and the max Q14
relative error over whole [row, N] distance rows (shard_dist) of the sampled queries.

usage: python scripts/diag_chain_err.py [c2|c3|c4|small|medium ...]   (KGQ_LIB_PATH selects a build)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import synth  # noqa: E402
from paper_2503_02172_b200 import Engine  # noqa: E402

CFG = {  # name: (model, N, R, d, H, B, structures, table seed, rows sampled)
    "c2": ("betae", 14505, 237, 400, 1600, 1024, synth.ALL_STRUCTURES, 2503_02172 + 1, 3),
    "c3": ("q2b", 63361, 200, 400, 1600, 1024, synth.EPFO, 2503_02172 + 2, 2),
    "c4": ("betae", 14951, 1345, 400, 1600, 4096, synth.NEGATION, 2503_02172 + 3, 3),
    "small": ("betae", 1000, 20, 40, 96, 37, synth.ALL_STRUCTURES, 21, 37),
    "small_spread": ("betae", 1000, 20, 40, 96, 37, synth.ALL_STRUCTURES, 21, 37, "spread"),
    "gqe_spread": ("gqe", 1000, 20, 40, 96, 37, synth.EPFO, 21, 37, "spread"),
    "q2b_spread": ("q2b", 1000, 20, 40, 96, 37, synth.EPFO, 21, 37, "spread"),
    "gqe_small": ("gqe", 1000, 20, 40, 96, 37, synth.EPFO, 21, 37),
    "q2b_small": ("q2b", 1000, 20, 40, 96, 37, synth.EPFO, 21, 37),
    "medium": ("betae", 3000, 40, 128, 512, 300, synth.ALL_STRUCTURES, 21, 40),
}


def run(name):
    model, N, R, d, H, B, structs, seed, nrows = CFG[name][:9]
    dist = CFG[name][9] if len(CFG[name]) > 9 else "kgr-init"
    t = synth.make_tables(model, N, R, d, hidden=H, seed=seed, dist=dist)
    e = Engine(model, N, R, d, hidden=H, max_batch=B, max_k=16)
    e.load_tables(t)
    m = O.Model(model, t, dim=d)
    rng = np.random.default_rng(0)
    res = {}
    for s in structs:
        a, r = synth.make_queries(s, B, N, R, seed=synth.query_seed(seed, s))
        rows = np.unique(np.r_[rng.choice(B, size=min(B, nrows) - 1, replace=False), B - 1])
        da, dr = torch.from_numpy(a).cuda(), torch.from_numpy(r).cuda()
        qe = e.query_embedding(s, da, dr).cpu().numpy()[rows].astype(np.float64)
        _, _, sd = e.submit(s, da, dr, 10, shard_dist=True)
        sd = sd.cpu().numpy()[rows].astype(np.float64)
        ref_q = m.query_embedding(s, a[rows], r[rows])
        ref_d = m.scores(s, a[rows], r[rows])
        out = {}
        for f in (1e-2, 1e-3):
            floor = f * np.max(np.abs(ref_q), axis=-1, keepdims=True)
            out[f"chain_floor{f:g}"] = float((np.abs(qe - ref_q) / np.maximum(np.abs(ref_q), floor)).max())
        s_q = 1e-3 * np.median(ref_d, axis=-1, keepdims=True)
        out["dist"] = float((np.abs(sd - ref_d) / np.maximum(np.abs(ref_d), s_q)).max())
        res[s] = out
    e.close()
    print(json.dumps({"config": name, "lib": os.environ.get("KGQ_LIB_PATH", "default"), "rows": int(nrows),
                      "errors": res}), flush=True)


if __name__ == "__main__":
    for n in (sys.argv[1:] or ["small", "medium", "c2", "c4", "c3"]):
        run(n)
