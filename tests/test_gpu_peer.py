"""N2: the cross-shard all-gather fused into the top-k kernel over peer memory
(kgq_set_peers / kgq_merge_peers, csrc/peer.cu).  W virtual ranks on one GPU: every rank's
peer buffer is ordinary device memory and the push / flag / merge protocol runs exactly as over
NVLink (the kernels only see device pointers).  The merged global top-k must equal the
single-shard top-k bit for bit, across epochs (parity double-buffering), graph replays, the
fused (k <= 32 BetaE) and separate push kernels, and mixed batches."""
import os

import numpy as np
import pytest
import torch

import oracle as O
import synth
from parity import assert_topk_ok

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2503_02172_b200 import Engine, KgqError  # noqa: E402

N, R, D, H = 1000, 20, 40, 96


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.int32)).cuda()


def peer_ranks(model, t, W, max_batch=64, max_k=64):
    engs = [Engine(model, N, R, D, hidden=H, max_batch=max_batch, max_k=max_k, world_size=W, rank=r)
            for r in range(W)]
    for e in engs:
        e.load_tables(t)
    bufs = [torch.empty(engs[0].peer_bytes(W), dtype=torch.uint8, device="cuda") for _ in range(W)]
    for r, e in enumerate(engs):
        e.set_peers(r, W, [b.data_ptr() for b in bufs])
    return engs, bufs


@pytest.mark.parametrize("model,structs,ks", [("betae", ("1p", "2u", "pin"), (16, 40)),
                                              ("gqe", ("2p", "up"), (10,))])
def test_peer_merge_equals_single_gpu(model, structs, ks):
    t = synth.make_tables(model, N, R, D, hidden=H, seed=5)
    full = Engine(model, N, R, D, hidden=H, max_batch=64, max_k=64)
    full.load_tables(t)
    m = O.Model(model, t, dim=D)
    for W in (2, 3, 8):
        engs, bufs = peer_ranks(model, t, W)
        for s in structs:
            for k in ks:
                # same input tensors every round: the 2nd submit captures a graph, the 3rd and
                # 4th replay it (the epoch bump and the push run inside the graph)
                a0, r0 = synth.make_queries(s, 33, N, R, seed=3)
                da, dr = dev(a0), dev(r0)
                for rnd in range(4):
                    a, r = synth.make_queries(s, 33, N, R, seed=100 + rnd)
                    da.copy_(dev(a))
                    dr.copy_(dev(r))
                    fd, fi = full.submit(s, da, dr, k)
                    local = [e.submit(s, da, dr, k) for e in engs]   # push to every rank
                    merged = [e.merge_peers(33, k) for e in engs]      # wait + merge on every rank
                    torch.cuda.synchronize()
                    if rnd == 0 or W == 3:  # the merged lists against the oracle (Q15)
                        ref = m.scores(s, a, r)
                        mdn, min_ = merged[-1][0].cpu().numpy(), merged[-1][1].cpu().numpy()
                        for b in range(33):
                            assert_topk_ok(mdn[b], min_[b], ref[b], k, what=f"p2p W={W} {s} k={k} row {b}")
                    for rank, (md, mi) in enumerate(merged):
                        assert torch.equal(mi, fi), (model, s, k, W, rnd, rank)
                        assert torch.equal(md, fd), (model, s, k, W, rnd, rank)
                    # the local (shard) outputs are still written
                    ld, li = local[0]
                    assert torch.all((li >= engs[0].shard[0]) & (li < engs[0].shard[1]))
        for e in engs:
            e.check_errors()
            e.close()
    full.close()


def test_peer_mixed_batch_and_invalid_rows():
    t = synth.make_tables("betae", N, R, D, hidden=H, seed=5)
    groups = []
    for i, s in enumerate(("2p", "up", "3in", "2u-DM")):
        a, r = synth.make_queries(s, 9 + i, N, R, seed=40 + i)
        if i == 1:
            a[3, 0] = N  # out-of-range anchor: NaN / -1 row on every rank, merged as such
        groups.append((s, dev(a), dev(r)))
    Q = sum(int(g[1].shape[0]) for g in groups)
    full = Engine("betae", N, R, D, hidden=H, max_batch=128, max_k=32)
    full.load_tables(t)
    fd, fi = full.submit_mixed(groups, 12)
    m = O.Model("betae", t, dim=D)
    with pytest.raises(KgqError, match="ERANGE"):
        full.check_errors()
    engs, bufs = peer_ranks("betae", t, 3, max_batch=128, max_k=32)
    for e in engs:
        e.submit_mixed(groups, 12)
    merged = [e.merge_peers(Q, 12) for e in engs]
    torch.cuda.synchronize()
    for md, mi in merged:
        assert torch.equal(mi, fi)
        assert torch.equal(torch.nan_to_num(md, nan=-7.0), torch.nan_to_num(fd, nan=-7.0))
    bad = 9 + 3
    assert torch.all(mi[bad] == -1) and torch.all(torch.isnan(md[bad]))
    mdn, min_ = md.cpu().numpy(), mi.cpu().numpy()
    q = 0
    for s, a, r in groups:   # every valid merged row against the oracle (Q15)
        an, rn = a.cpu().numpy(), r.cpu().numpy()
        ok = [b for b in range(an.shape[0]) if q + b != bad]
        ref = m.scores(s, an[ok], rn[ok])
        for j, b in enumerate(ok):
            assert_topk_ok(mdn[q + b], min_[q + b], ref[j], 12, what=f"p2p mixed {s} row {b}")
        q += an.shape[0]
    for e in engs:
        with pytest.raises(KgqError, match="ERANGE"):
            e.check_errors()
        e.close()
    full.close()


def test_peer_missing_rank_times_out_instead_of_hanging():
    """A rank that never pushes: the merge times out (no GPU hang), its rows are NaN / -1, the
    session is poisoned on every rank (later merges fail loudly instead of pairing lists of
    different submits), and kgq_set_peers on every rank restores it."""
    t = synth.make_tables("betae", N, R, D, hidden=H, seed=5)
    os.environ["KGQ_PEER_TIMEOUT_MS"] = "200"
    try:
        engs, bufs = peer_ranks("betae", t, 2)
    finally:
        del os.environ["KGQ_PEER_TIMEOUT_MS"]
    a, r = synth.make_queries("1p", 20, N, R, seed=3)
    engs[0].submit("1p", dev(a), dev(r), 10)  # rank 1 never pushes
    md, mi = engs[0].merge_peers(20, 10)
    torch.cuda.synchronize()
    with pytest.raises(KgqError, match="rank 1 did not publish"):
        engs[0].check_errors()
    assert torch.all(mi == -1) and torch.all(torch.isnan(md))
    # both ranks push and merge now, but the session stays closed on both
    for e in engs:
        e.submit("1p", dev(a), dev(r), 10)
    outs = [e.merge_peers(20, 10) for e in engs]
    torch.cuda.synchronize()
    for e, (md, mi) in zip(engs, outs):
        assert torch.all(mi == -1)
        with pytest.raises(KgqError, match="closed by an earlier timeout"):
            e.check_errors()
    # re-registration on every rank reopens it
    for rk, e in enumerate(engs):
        e.set_peers(rk, 2, [b.data_ptr() for b in bufs])
    full = Engine("betae", N, R, D, hidden=H, max_batch=64, max_k=64)
    full.load_tables(t)
    fd, fi = full.submit("1p", dev(a), dev(r), 10)
    for e in engs:
        e.submit("1p", dev(a), dev(r), 10)
    outs = [e.merge_peers(20, 10) for e in engs]
    torch.cuda.synchronize()
    for e, (md, mi) in zip(engs, outs):
        e.check_errors()
        assert torch.equal(mi, fi) and torch.equal(md, fd)
    for e in engs + [full]:
        e.close()


def test_peer_push_and_merge_are_paired():
    """A second pushing submit before the merge, or a merge without a push, is rejected
    (KGQ_ESTATE) instead of racing a peer's read of the same slot."""
    t = synth.make_tables("gqe", N, R, D, hidden=H, seed=5)
    engs, bufs = peer_ranks("gqe", t, 2)
    a, r = synth.make_queries("1p", 8, N, R, seed=1)
    with pytest.raises(KgqError, match="no pushing submit"):
        engs[0].merge_peers(8, 5)
    engs[0].submit("1p", dev(a), dev(r), 5)
    with pytest.raises(KgqError, match="has not been merged"):
        engs[0].submit("1p", dev(a), dev(r), 5)
    with pytest.raises(KgqError, match="has not been merged"):
        engs[0].submit_host("1p", a, r, 5)
    with pytest.raises(KgqError, match="has not been merged"):
        engs[0].submit_mixed([("1p", dev(a), dev(r))], 5)
    engs[1].submit("1p", dev(a), dev(r), 5)
    m0 = engs[0].merge_peers(8, 5)
    m1 = engs[1].merge_peers(8, 5)
    torch.cuda.synchronize()
    for e in engs:
        e.check_errors()
    assert torch.equal(m0[1], m1[1])
    for e in engs:
        e.close()


def test_peer_argument_errors():
    t = synth.make_tables("gqe", N, R, D, hidden=H, seed=5)
    e = Engine("gqe", N, R, D, hidden=H, max_batch=16, max_k=16)
    e.load_tables(t)
    with pytest.raises(KgqError, match="ESTATE"):
        e.merge_peers(4, 5)  # no peers registered
    buf = torch.empty(e.peer_bytes(2) + 512, dtype=torch.uint8, device="cuda")
    p = buf.data_ptr()
    with pytest.raises(KgqError, match="EINVAL"):
        e.set_peers(0, 9, [p] * 9)  # world > 8
    with pytest.raises(KgqError, match="EINVAL"):
        e.set_peers(2, 2, [p, p])  # rank >= world
    with pytest.raises(KgqError, match="aligned"):
        e.set_peers(0, 2, [p + 8, p])
    with pytest.raises(KgqError):
        e.peer_bytes(0)
    e.set_peers(0, 1, [p])  # a world of one: push to itself, merge == local top-k
    a, r = synth.make_queries("1p", 4, N, R, seed=1)
    ld, li = e.submit("1p", dev(a), dev(r), 5)
    md, mi = e.merge_peers(4, 5)
    assert torch.equal(mi, li) and torch.equal(md, ld)
    e.set_peers(0, 0, [])  # off again
    with pytest.raises(KgqError, match="ESTATE"):
        e.merge_peers(4, 5)
    e.close()
