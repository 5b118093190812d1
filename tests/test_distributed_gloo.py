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


def _rank_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N, R, d = 157, 5, 8
        t = synth.make_tables("q2b", N, R, d, seed=6)
        m = O.Model("q2b", t, dim=d)
        a, r = synth.make_queries("2u", 5, N, R, seed=2)
        full = m.scores("2u", a, r)
        rng = np.random.default_rng(0)
        answers = [rng.choice(N, size=4, replace=False) for _ in range(5)]
        lo, hi = kgq.shard_range(N, world, rank)
        # phase 1 (KGQ_RANK_DIST): distances of the answers this shard owns, +inf elsewhere
        ad = torch.full((5, 4), float("inf"), dtype=torch.float64)
        for b in range(5):
            for j, e in enumerate(answers[b]):
                if lo <= e < hi:
                    ad[b, j] = full[b, e]
        dist.all_reduce(ad, op=dist.ReduceOp.MIN)
        # phase 2 (KGQ_RANK_COUNT): better non-answers inside this shard, summed over ranks
        cnt = torch.zeros((5, 4), dtype=torch.int64)
        for b in range(5):
            ans = set(int(x) for x in answers[b])
            for j, e in enumerate(answers[b]):
                for x in range(lo, hi):
                    if x not in ans and (full[b, x] < ad[b, j] or (full[b, x] == ad[b, j] and x < e)):
                        cnt[b, j] += 1
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
        ok = all(O.filtered_ranks(full[b], answers[b])[int(e)] == 1 + int(cnt[b, j])
                 for b in range(5) for j, e in enumerate(answers[b]))
        q.put((rank, ok))
    except Exception as e:
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_two_phase_filtered_rank_protocol_over_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


def _query_split_worker(rank, world, port, q):
    """Query-split data plane (kgq_comm_init KGQ_SPLIT_QUERIES) on CPU: the replicated batch's
    rows kgq_query_range(B, W, r) run on rank r (the oracle stands in for the GPU path), each rank
    contributes ceil(B / W) rows (padded: NaN / -1) to one all-gather, and the first B gathered
    rows are the whole batch's top-k -- the same steps and buffer layout as submit_comm."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N, R, d, k = 211, 6, 8, 7
        t = synth.make_tables("betae", N, R, d, hidden=16, seed=9)
        m = O.Model("betae", t, dim=d)
        out = {}
        for s, B in (("2p", 11), ("up", 3), ("inp", 1)):
            a, r = synth.make_queries(s, B, N, R, seed=13)   # replicated on every rank
            lo, hi = kgq.query_range(B, world, rank)
            c = -(-B // world)
            send_d = torch.full((c, k), float("nan"), dtype=torch.float64)
            send_i = torch.full((c, k), -1, dtype=torch.int64)
            if hi > lo:
                ld, li = O.topk(m.scores(s, a[lo:hi], r[lo:hi]), k)
                send_d[: hi - lo] = torch.from_numpy(ld)
                send_i[: hi - lo] = torch.from_numpy(li)
            gd = torch.empty((world * c, k), dtype=torch.float64)
            gi = torch.empty((world * c, k), dtype=torch.int64)
            dist.all_gather_into_tensor(gd, send_d)
            dist.all_gather_into_tensor(gi, send_i)
            out[s] = (gd[:B].numpy(), gi[:B].numpy())
        q.put((rank, out))
    except Exception as e:
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_query_split_protocol_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_query_split_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for v in res.values():
        assert not isinstance(v, str), v
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    N, R, d, k = 211, 6, 8, 7
    t = synth.make_tables("betae", N, R, d, hidden=16, seed=9)
    m = O.Model("betae", t, dim=d)
    for s, B in (("2p", 11), ("up", 3), ("inp", 1)):
        a, r = synth.make_queries(s, B, N, R, seed=13)
        gd, gi = O.topk(m.scores(s, a, r), k)
        for rank in range(world):
            md, mi = res[rank][s]
            np.testing.assert_array_equal(mi, gi)
            # fp64 BLAS groups the MLP sums differently for a row slice than for the batch
            np.testing.assert_allclose(md, gd, rtol=1e-12)
