"""Small workload for compute-sanitizer (scripts/sanitize.sh): every kernel family of libkgq.so
once, on sizes the sanitizers finish in minutes.  Prints one line per case; exits non-zero if a
result is wrong (the sanitizer's own report is the evidence)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2503_02172_b200 import Engine  # noqa: E402
from paper_2503_02172_b200.sharded import answers_csr  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.int32)).cuda()


def case(name, fn):
    fn()
    torch.cuda.synchronize()
    print(f"case {name}: ok", flush=True)


# BetaE with split-K tails (K = 256 / 512 > one split), tensor-core scorer, block-minima top-k
N, R, d, H, B = 3000, 40, 128, 512, 300
t = synth.make_tables("betae", N, R, d, hidden=H, seed=21)
e = Engine("betae", N, R, d, hidden=H, max_batch=320, max_k=16)
e.load_tables(t)
for s in ("1p", "3in", "up", "pni"):
    a, r = synth.make_queries(s, B, N, R, seed=3)
    case(f"betae {s} split-K", lambda: e.submit(s, dev(a), dev(r), 10))
groups = [(s, dev(a), dev(r)) for s, (a, r) in
          ((s, synth.make_queries(s, 20 + 3 * i, N, R, seed=40 + i)) for i, s in enumerate(("2p", "ip", "2u-DM")))]
case("betae mixed", lambda: e.submit_mixed(groups, 10))
# fused top-k (per-stripe lists in the scorer epilogue + list merge): forced ON, many stripes
e.set_fused_topk("on")
for s in ("1p", "up"):
    a, r = synth.make_queries(s, B, N, R, seed=5)
    case(f"betae {s} fused top-k", lambda: e.submit(s, dev(a), dev(r), 10))
case("betae mixed fused top-k", lambda: e.submit_mixed(groups, 10))
e.set_fused_topk("auto")
e.check_errors()
e.close()

# N2 peer protocol: three virtual ranks, push + merge
N2, R2, d2, H2 = 1000, 20, 40, 96
t2 = synth.make_tables("betae", N2, R2, d2, hidden=H2, seed=5)
W = 3
engs = [Engine("betae", N2, R2, d2, hidden=H2, max_batch=64, max_k=32, world_size=W, rank=rk) for rk in range(W)]
for x in engs:
    x.load_tables(t2)
bufs = [torch.empty(engs[0].peer_bytes(W), dtype=torch.uint8, device="cuda") for _ in range(W)]
for rk, x in enumerate(engs):
    x.set_peers(rk, W, [b.data_ptr() for b in bufs])
a, r = synth.make_queries("2u", 33, N2, R2, seed=3)


def peer_round():
    for x in engs:
        x.submit("2u", dev(a), dev(r), 16)
    for x in engs:
        x.merge_peers(33, 16)


case("peer push / merge", peer_round)
for x in engs:
    x.check_errors()
    x.close()

# GQE / Q2B SIMT scorers: tiled (B 40) and streamed (B 4), filtered rank
for model in ("gqe", "q2b"):
    t3 = synth.make_tables(model, 5000, 20, 64, seed=8)
    g = Engine(model, 5000, 20, 64, max_batch=64, max_k=16)
    g.load_tables(t3)
    for Bq in (40, 4):
        a, r = synth.make_queries("up", Bq, 5000, 20, seed=9)
        case(f"{model} up B {Bq}", lambda: g.submit("up", dev(a), dev(r), 10))
    a, r = synth.make_queries("2p", 8, 5000, 20, seed=1)
    off, ids = answers_csr([np.arange(i, 40 + i, 7) for i in range(8)])
    case(f"{model} filtered rank", lambda: g.rank_answers("2p", dev(a), dev(r), dev(off), dev(ids), 3))
    g.check_errors()
    g.close()
print("all cases done")
