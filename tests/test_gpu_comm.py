"""The library's own NCCL communicator (kgq_comm_init) on one GPU: a world of
one rank runs the real NCCL calls (unique id, ncclCommInitRank, the all-gather group, the
all-reduces of the filtered rank, ncclCommGetAsyncError) through the exact code paths of a W-rank
job -- the merge of one list, the reassembly of one row slice.  Results must equal the plain
submit bit for bit and match the oracle.  The W > 1 protocols (row partition, padded
all-gather, merge, two-phase rank) are covered over gloo in test_distributed_gloo.py."""
import numpy as np
import pytest

import oracle as O
import synth
from parity import assert_topk_ok

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)
from paper_2503_02172_b200 import Engine, KgqError  # noqa: E402
from paper_2503_02172_b200.kgq import (RANK_FILTERED, SPLIT_ENTITIES, SPLIT_QUERIES,  # noqa: E402
                                       nccl_unique_id)
from paper_2503_02172_b200.sharded import answers_csr  # noqa: E402

N, R, D, H = 1000, 20, 40, 96


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.int32)).cuda()


@pytest.mark.parametrize("split", [SPLIT_ENTITIES, SPLIT_QUERIES])
def test_comm_world_one_equals_plain_submit(split):
    t = synth.make_tables("betae", N, R, D, hidden=H, seed=5)
    plain = Engine("betae", N, R, D, hidden=H, max_batch=64, max_k=16)
    plain.load_tables(t)
    e = Engine("betae", N, R, D, hidden=H, max_batch=64, max_k=16)
    e.load_tables(t)
    e.comm_init(nccl_unique_id(), 1, 0, split)
    m = O.Model("betae", t, dim=D)
    for s in ("1p", "2u", "pni", "up-DM"):
        a, r = synth.make_queries(s, 33, N, R, seed=3)
        for rnd in range(3):  # the 2nd identical submit is captured into a graph, the 3rd replays it
            pd, pi = plain.submit(s, dev(a), dev(r), 12)
            cd, ci = e.submit(s, dev(a), dev(r), 12)
            torch.cuda.synchronize()
            assert torch.equal(ci, pi) and torch.equal(cd, pd), (s, rnd)
        ref = m.scores(s, a, r)
        for b in range(33):
            assert_topk_ok(cd[b].cpu().numpy(), ci[b].cpu().numpy(), ref[b], 12, what=f"comm {s} row {b}")
        hd, hi = e.submit_host(s, a, r, 12)
        np.testing.assert_array_equal(hi, pi.cpu().numpy())
    groups = [(s, dev(a), dev(r)) for s, (a, r) in
              ((s, synth.make_queries(s, 7 + i, N, R, seed=40 + i)) for i, s in enumerate(("2p", "up", "3in")))]
    md, mi = e.submit_mixed(groups, 10)
    pd, pi = plain.submit_mixed(groups, 10)
    torch.cuda.synchronize()
    assert torch.equal(mi, pi) and torch.equal(md, pd)
    e.check_errors()  # also polls ncclCommGetAsyncError
    with pytest.raises(KgqError, match="ESTATE"):
        e.comm_init(nccl_unique_id(), 1, 0, split)  # one communicator per context
    if split == SPLIT_QUERIES:
        with pytest.raises(KgqError, match="shard_dist"):
            e.submit("1p", dev(a[:, :1]), dev(r[:, :1]), 5, shard_dist=True)
    e.comm_destroy()
    ld, li = e.submit("1p", dev(a[:, :1]), dev(r[:, :1]), 5)
    torch.cuda.synchronize()
    e.close()
    plain.close()


def test_comm_filtered_rank_and_metrics():
    """KGQ_RANK_FILTERED through the communicator (two phases + all-reduces inside) and the
    MRR / Hits kernel, against the oracle's filtered ranks and mrr_hits (N1)."""
    t = synth.make_tables("gqe", N, R, D, hidden=H, seed=8)
    e = Engine("gqe", N, R, D, hidden=H, max_batch=64, max_k=16)
    e.load_tables(t)
    e.comm_init(nccl_unique_id(), 1, 0, SPLIT_ENTITIES)
    m = O.Model("gqe", t, dim=D)
    rng = np.random.default_rng(3)
    a, r = synth.make_queries("2p", 21, N, R, seed=5)
    ref = m.scores("2p", a, r)
    lists = [np.unique(np.r_[np.argsort(ref[b])[: rng.integers(0, 3)], rng.choice(N, 4, replace=False)])
             for b in range(21)]
    off, ids = answers_csr(lists)
    hard = (rng.random(len(ids)) < 0.7).astype(np.uint8)
    _, ranks = e.rank_answers("2p", dev(a), dev(r), dev(off), dev(ids), RANK_FILTERED)
    ranks_h = ranks.cpu().numpy()
    per_q = []
    for b in range(21):
        exact = O.filtered_ranks(ref[b], lists[b])
        keep = np.setdiff1d(np.arange(N), lists[b])
        for j in range(off[b], off[b + 1]):
            da, tol = ref[b, ids[j]], 1e-4 * ref[b, ids[j]]
            lo = 1 + int(np.count_nonzero(ref[b, keep] < da - tol))   # Q15: ties within 1e-4
            hi = 1 + int(np.count_nonzero(ref[b, keep] <= da + tol))
            assert lo <= ranks_h[j] <= hi and lo <= exact[int(ids[j])] <= hi, (b, j)
        hr = [int(ranks_h[j]) for j in range(off[b], off[b + 1]) if hard[j]]
        if hr:
            per_q.append(O.mrr_hits(hr))
    met = e.rank_metrics(dev(off), ranks, torch.from_numpy(hard).cuda()).cpu().numpy()
    np.testing.assert_allclose(met[:4], np.mean(per_q, axis=0), rtol=1e-12)
    assert met[4] == len(per_q)
    e.close()
