"""N > 1 host path on CPU: world_size 2 (and 3) gloo process groups.

Each rank takes its entity shard from the C library's kgq_shard_range, computes its local
top-k (global ids) -- on CPU here the oracle stands in for the GPU scorer, which the GPU
tests cover -- exchanges it with the product's all_gather_topk helper over gloo, and merges.
The merged result must equal the single-process global top-k exactly, on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth

kgq = pytest.importorskip("paper_2503_02172_b200.kgq")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_02172_b200.sharded import all_gather_topk
        N, R, d, k = 301, 7, 12, 9
        t = synth.make_tables("betae", N, R, d, hidden=16, seed=4)
        m = O.Model("betae", t, dim=d)
        out = {}
        for s in ("1p", "2u", "pni"):
            a, r = synth.make_queries(s, 6, N, R, seed=8)
            lo, hi = kgq.shard_range(N, world, rank)          # the C ABI's partition
            dist_rows = m.scores(s, a, r, rows=np.arange(lo, hi))
            ld, li = O.topk(dist_rows, k, ids=np.arange(lo, hi))
            gd, gi = all_gather_topk(torch.from_numpy(ld), torch.from_numpy(li))
            assert gd.shape == (world, 6, k)
            md, mi = O.merge_topk(list(gd.numpy()), list(gi.numpy()), k)
            out[s] = (md, mi)
        q.put((rank, out))
    except Exception as e:  # surface the failure instead of timing out
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_topk_over_gloo_equals_global(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for v in res.values():
        assert not isinstance(v, str), v
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    N, R, d, k = 301, 7, 12, 9
    t = synth.make_tables("betae", N, R, d, hidden=16, seed=4)
    m = O.Model("betae", t, dim=d)
    for s in ("1p", "2u", "pni"):
        a, r = synth.make_queries(s, 6, N, R, seed=8)
        gd, gi = O.topk(m.scores(s, a, r), k)
        for rank in range(world):
            md, mi = res[rank][s]
            np.testing.assert_array_equal(mi, gi)
            np.testing.assert_array_equal(md, gd)


def test_shard_ranges_cover_and_balance():
    for n in (10, 14505, 2_000_000):
        for w in (2, 4, 8):
            rs = [kgq.shard_range(n, w, r) for r in range(w)]
            sizes = [b - a for a, b in rs]
            assert sum(sizes) == n and max(sizes) - min(sizes) <= -(-n // w)
