"""GPU parity: the CUDA path (through the C ABI) vs the float64 oracle, element by element.

Sizes span several tiles with ragged tails (entities not a multiple of 128, dims not a
multiple of 16, batches not a multiple of the 64-row tile), both input recipes, every
structure of every model, plus edge cases.  Full-size configs are in test_gpu_fullsize.py.
"""
import numpy as np
import pytest

import oracle as O
import synth
from parity import (assert_dist_close, assert_embedding_close, assert_topk_ok, chain_tolerance)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)
from paper_2503_02172_b200 import Engine, KgqError  # noqa: E402

STRUCTS = {"gqe": synth.EPFO, "q2b": synth.EPFO, "betae": synth.ALL_STRUCTURES}
SMALL = dict(N=1000, R=20, d=40, H=96, B=37)  # ragged everywhere


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


_engines = {}


def engine(model, dist="kgr-init", N=SMALL["N"], R=SMALL["R"], d=SMALL["d"], H=SMALL["H"],
           layers=2, terminal="regularizer", max_batch=64, max_k=32, seed=21):
    key = (model, dist, N, R, d, H, layers, terminal, max_batch, max_k, seed)
    if key not in _engines:
        t = synth.make_tables(model, N, R, d, hidden=H, n_layers=layers, seed=seed, dist=dist)
        e = Engine(model, N, R, d, hidden=H, n_hidden_layers=layers, terminal=terminal,
                   max_batch=max_batch, max_k=max_k)
        e.load_tables(t)
        _engines[key] = (e, O.Model(model, t, dim=d, n_layers=layers,
                                    terminal=O.TERMINAL_SOFTMAX if terminal == "softmax"
                                    else O.TERMINAL_REGULARIZER), t)
    return _engines[key]


def run_case(model, s, dist="kgr-init", B=SMALL["B"], k=10, **kw):
    terminal = kw.get("terminal", "regularizer")
    e, m, t = engine(model, dist, **kw)
    N = t["entity"].shape[0]
    R = t["relation"].shape[0]
    a, r = synth.make_queries(s, B, N, R, seed=synth.query_seed(7, s))
    td, ti, sd = e.submit(s, dev(a), dev(r), k, shard_dist=True)
    e.check_errors()
    ref = m.scores(s, a, r)
    assert_dist_close(sd.cpu().numpy(), ref, what=f"{model} {s} dist")   # north_star: 1e-4
    td, ti = td.cpu().numpy(), ti.cpu().numpy()
    for b in range(B):
        assert_topk_ok(td[b], ti[b], ref[b], k, what=f"{model} {s} row {b}")
    qe = e.query_embedding(s, dev(a), dev(r)).cpu().numpy()
    ref_q = m.query_embedding(s, a, r)
    assert_embedding_close(qe, ref_q, rel=chain_tolerance(s, dist, model, terminal), what=f"{model} {s} chain")
    return e


@pytest.mark.parametrize("s", ["1p", "3in", "up"])
def test_betae_medium_dims_split_k_plans(s):
    """K = 256-512 and 300 queries: the planner's split-K tails (publish / last-arriver reduce),
    BN = 160 / 192 tiles and multi-M-pair grids run here (the SMALL config has K <= 120, one
    K-split); distances, top-k and chain vs the oracle."""
    run_case("betae", s, B=300, k=10, N=3000, R=40, d=128, H=512, max_batch=320)


@pytest.mark.parametrize("s", ["1p", "2p", "2i"])
def test_toy_gqe_config(s):
    # BASELINE.json configs[0]: GQE 1p/2p/2i on a toy KG, 200 entities, 10 rels, dim 32, B 16
    run_case("gqe", s, N=200, R=10, d=32, H=8, B=16, k=10, max_batch=16, max_k=10)


@pytest.mark.parametrize("model", ["gqe", "q2b", "betae"])
@pytest.mark.parametrize("dist", ["kgr-init", "spread"])
def test_every_structure(model, dist):
    for s in STRUCTS[model]:
        run_case(model, s, dist)


def test_betae_softmax_terminal_flag():
    for s in ("1p", "2in", "ip", "up"):
        run_case("betae", s, terminal="softmax")


def test_betae_three_hidden_layers():
    run_case("betae", "3p", layers=3)
    run_case("betae", "pni", layers=1)


def test_betae_entity_terms_definition():
    """C/U/V planes reproduce the literal KL: KL(e||q) = lnB(q) + C + a_q U + b_q V."""
    e, m, t = engine("betae", "spread")
    cuv = e.entity_terms().cpu().numpy().astype(np.float64)  # [3, d, N]
    d = SMALL["d"]
    ent = m.entity_view()
    rng = np.random.default_rng(0)
    q = rng.uniform(0.05, 5, size=(5, 2 * d))
    for i in range(5):
        lit = O.kl_beta(ent[:, :d], ent[:, d:], q[i, :d], q[i, d:])               # [N, d]
        dec = O.log_beta(q[i, :d], q[i, d:]) + cuv[0].T + q[i, :d] * cuv[1].T + q[i, d:] * cuv[2].T
        np.testing.assert_allclose(dec, lit, rtol=1e-5, atol=2e-6 * np.abs(cuv).max())


def test_planted_kg_answers_exact():
    from planted import PlantedKG
    from test_oracle_planted import planted_queries
    kg = PlantedKG(n_entity=200, n_relation=12, dim=32, depth=4, seed=7)
    t = synth.make_tables("gqe", kg.n, 12, 32, seed=1)
    t["entity"], t["relation"] = kg.E.copy(), kg.R.copy()
    e = Engine("gqe", kg.n, 12, 32, max_batch=16, max_k=8)
    e.load_tables(t)
    for s in ("1p", "2p", "3p", "2i", "3i", "2u", "up"):
        a, r = planted_queries(kg, s, 12, seed=hash(s) % 1000)
        td, ti = e.submit(s, dev(a), dev(r), 4)
        td, ti = td.cpu().numpy(), ti.cpu().numpy()
        for b in range(len(a)):
            ans = sorted(kg.answers(s, list(a[b]), list(r[b])))
            n = len(ans)
            assert list(ti[b, :n]) == ans, (s, b)
            if s in ("1p", "2p", "3p", "2u", "up"):   # pure translations: exact in fp32
                assert np.all(td[b, :n] == 0)
            assert td[b, n] > 0.5


def test_virtual_shards_merge_equals_single_gpu():
    """Entity sharding (§8(e)) with W contexts on one GPU + kgq_merge_topk == 1 shard."""
    N, R, d = 1000, 20, 40
    t = synth.make_tables("betae", N, R, d, hidden=96, seed=5)
    full = Engine("betae", N, R, d, hidden=96, max_batch=64, max_k=32)
    full.load_tables(t)
    m = O.Model("betae", t, dim=d)
    for s in ("1p", "2u", "pin"):
        a, r = synth.make_queries(s, 33, N, R, seed=3)
        fd, fi = full.submit(s, dev(a), dev(r), 16)
        ref = m.scores(s, a, r)
        for W in (2, 3, 8):
            parts = []
            for rank in range(W):
                e = Engine("betae", N, R, d, hidden=96, max_batch=64, max_k=32, world_size=W, rank=rank)
                e.load_tables(t)
                assert e.shard == O.shard_range(N, W, rank)
                parts.append(e.submit(s, dev(a), dev(r), 16))
                e.close()
            md, mi = full.merge_topk(torch.stack([p[0] for p in parts]),
                                     torch.stack([p[1] for p in parts]), 16)
            # the merged global top-k against the oracle (Q15; P:425 ranking), then bit-identity
            # with the one-shard path
            mdn, min_ = md.cpu().numpy(), mi.cpu().numpy()
            for b in range(33):
                assert_topk_ok(mdn[b], min_[b], ref[b], 16, what=f"merged W={W} {s} row {b}")
            assert torch.equal(mi, fi), (s, W)
            assert torch.equal(md, fd), (s, W)


def test_edge_cases():
    e, m, t = engine("gqe")
    a, r = synth.make_queries("2p", 5, SMALL["N"], SMALL["R"], seed=1)
    # empty batch: no-op
    z = torch.empty((0, 1), dtype=torch.int32, device="cuda")
    td, ti = e.submit("1p", z, z, 5)
    assert td.shape == (0, 5)
    # out-of-range anchor and relation -> NaN / -1 rows + KGQ_ERANGE
    bad_a, bad_r = a.copy(), r.copy()
    bad_a[2, 0] = SMALL["N"]
    bad_r[4, 1] = -1
    td, ti = e.submit("2p", dev(bad_a), dev(bad_r), 5)
    with pytest.raises(KgqError, match="ERANGE"):
        e.check_errors()
    e.check_errors()  # cleared
    td, ti = td.cpu().numpy(), ti.cpu().numpy()
    assert np.all(np.isnan(td[[2, 4]])) and np.all(ti[[2, 4]] == -1)
    ref = m.scores("2p", a[[0, 1, 3]], r[[0, 1, 3]])
    for j, b in enumerate((0, 1, 3)):
        assert_topk_ok(td[b], ti[b], ref[j], 5)
    # negation on GQE, bad k, bad batch, unknown structure
    with pytest.raises(KgqError, match="UNSUPPORTED"):
        e.submit("2in", dev(a[:, :1].repeat(2, 1)), dev(r[:, :2]), 5)
    with pytest.raises(KgqError, match="EINVAL"):
        e.submit("1p", dev(a[:, :1]), dev(r[:, :1]), 33)
    with pytest.raises(KgqError, match="EINVAL"):
        big = np.zeros((65, 1), np.int32)
        e.submit("1p", dev(big), dev(big), 5)
    with pytest.raises(KgqError, match="valid: 1p"):
        e.submit("5p", dev(a), dev(r), 5)


def test_k_extremes_and_tiny_tables():
    # k == max_k == 256 on a 300-entity table; N < one 128-entity tile; d = 4
    run_case("q2b", "up", N=300, R=5, d=12, H=8, B=3, k=256, max_batch=8, max_k=256)
    run_case("gqe", "1p", N=50, R=3, d=4, H=8, B=2, k=50, max_batch=4, max_k=64)
    run_case("betae", "3in", N=129, R=3, d=8, H=16, B=65, k=1, max_batch=65, max_k=4)


def test_max_batch_ragged_rows():
    # B == max_batch, union doubles rows (2*B not a multiple of 64)
    run_case("betae", "up", B=64, max_batch=64)
    run_case("gqe", "3i", B=64, max_batch=64)


def test_submit_host_matches_device_path():
    e, m, t = engine("betae")
    a, r = synth.make_queries("inp", 20, SMALL["N"], SMALL["R"], seed=9)
    hd, hi = e.submit_host("inp", a, r, 7)
    dd, di = e.submit("inp", dev(a), dev(r), 7)
    np.testing.assert_array_equal(hi, di.cpu().numpy())
    np.testing.assert_array_equal(hd, dd.cpu().numpy())
    assert e.last_launch_count() > 0
    # async variant: several structures enqueued back to back (pinned buffers), one sync
    outs = {}
    for s in ("inp", "2u", "3in"):
        a2, r2 = synth.make_queries(s, 20, SMALL["N"], SMALL["R"], seed=11)
        pa = torch.from_numpy(a2.astype(np.int32)).pin_memory()
        pr = torch.from_numpy(r2.astype(np.int32)).pin_memory()
        od = torch.empty((20, 7)).pin_memory()
        oi = torch.empty((20, 7), dtype=torch.int32).pin_memory()
        e.submit_host(s, pa.numpy(), pr.numpy(), 7, out=(od.numpy(), oi.numpy()), sync=False)
        outs[s] = (a2, r2, pa, pr, od, oi)
    torch.cuda.synchronize()
    for s, (a2, r2, pa, pr, od, oi) in outs.items():
        dd, di = e.submit(s, dev(a2), dev(r2), 7)
        np.testing.assert_array_equal(oi.numpy(), di.cpu().numpy())
        np.testing.assert_array_equal(od.numpy(), dd.cpu().numpy())


def test_deterministic_repeat():
    e, m, t = engine("q2b")
    a, r = synth.make_queries("ip", 37, SMALL["N"], SMALL["R"], seed=2)
    x = e.submit("ip", dev(a), dev(r), 10, shard_dist=True)
    y = e.submit("ip", dev(a), dev(r), 10, shard_dist=True)
    for u, v in zip(x, y):
        assert torch.equal(u, v)


@pytest.mark.parametrize("model", ["gqe", "q2b", "betae"])
def test_small_batch_stream_scorer_matches_tiled(model):
    """B*branches <= 16 takes the streaming (HBM-regime) scorer; for GQE/Q2B it evaluates the
    same per-(q, e, d) expression in the same order as the tiled kernel -> bit-identical rows;
    BetaE batches above 16 rows use the tensor-core scorer -> agreement within 1e-5."""
    e, m, t = engine(model)
    N, R = SMALL["N"], SMALL["R"]
    for s in ("1p", "2u", "ip"):
        a, r = synth.make_queries(s, 37, N, R, seed=31)
        big = e.submit(s, dev(a), dev(r), 10, shard_dist=True)[2].cpu()
        for B in (1, 2, 3, 5, 8):
            td, ti, sd = e.submit(s, dev(a[:B]), dev(r[:B]), 10, shard_dist=True)
            if model == "betae":   # large batches take the tensor-core scorer (score_tc.cu)
                assert_dist_close(sd.cpu().numpy(), big[:B].numpy(), rel=1e-5, what=f"{s} B={B}")
            else:
                assert torch.equal(sd.cpu(), big[:B]), (model, s, B)
        run_case(model, s, B=3)


def test_chunked_topk_long_rows():
    """Rows > 32k entities use the multi-CTA top-k (chunks + k_merge)."""
    for k in (10, 256):
        run_case("gqe", "2u", N=70001, R=5, d=8, H=8, B=3, k=k, max_batch=4, max_k=256)
    run_case("betae", "1p", N=40000, R=5, d=8, H=16, B=20, k=16, max_batch=32, max_k=16)


@pytest.mark.parametrize("model", ["gqe", "q2b", "betae"])
def test_cuda_graph_replay_matches_eager(model):
    """Same (structure, batch, k, buffers) twice -> captured into a CUDA graph; replays with
    new query contents in the same buffers must equal the eager result."""
    e, m, t = engine(model)
    N, R = SMALL["N"], SMALL["R"]
    for s in ("2p", "2u", "3i"):
        da = torch.empty((37, synth.N_ANCHORS[s]), dtype=torch.int32, device="cuda")
        dr = torch.empty((37, synth.N_RELS[s]), dtype=torch.int32, device="cuda")
        out = (torch.empty((37, 10), device="cuda"), torch.empty((37, 10), dtype=torch.int32, device="cuda"))
        for rep in range(4):  # eager, capture+launch, replay, replay
            a, r = synth.make_queries(s, 37, N, R, seed=100 + rep)
            da.copy_(dev(a))
            dr.copy_(dev(r))
            e.submit(s, da, dr, 10, out=out)
            ref_d, ref_i = e.submit(s, dev(a), dev(r), 10)   # fresh buffers: eager
            assert torch.equal(out[1], ref_i) and torch.equal(out[0], ref_d), (model, s, rep)
        e.profile(True)   # graphs captured with stage events report per-replay stage times
        for _ in range(3):
            e.submit(s, da, dr, 10, out=out)
        prof = e.profile_read()
        e.profile(False)
        assert prof["score"][1] >= 3 and prof["score"][0] > 0


def _rank_bounds(ref_row, answers, rel=1e-4):
    """Oracle filtered rank interval under the Q14 tolerance (near-ties may flip)."""
    s_q = 1e-3 * np.median(ref_row)
    ans = set(int(a) for a in answers)
    keep = np.array([e not in ans for e in range(len(ref_row))])
    d = ref_row[keep]
    out = {}
    for a in ans:
        tol = rel * max(ref_row[a], s_q)
        out[a] = (1 + int(np.sum(d < ref_row[a] - tol)), 1 + int(np.sum(d <= ref_row[a] + tol)))
    return out


@pytest.mark.parametrize("model", ["gqe", "q2b", "betae"])
def test_filtered_ranks_n1(model):
    from paper_2503_02172_b200.sharded import answers_csr
    e, m, t = engine(model)
    N, R = SMALL["N"], SMALL["R"]
    rng = np.random.default_rng(5)
    for s in ("1p", "2u", "ip"):
        a, r = synth.make_queries(s, 37, N, R, seed=77)
        ref = m.scores(s, a, r)
        # answers: some of the true nearest (ranked well) + random entities
        lists = []
        for b in range(37):
            near = np.argsort(ref[b])[: rng.integers(0, 4)]
            rand = rng.choice(N, size=rng.integers(1, 6), replace=False)
            lists.append(np.unique(np.r_[near, rand]))
        off, ids = answers_csr(lists)
        ad, cnt = e.rank_answers(s, dev(a), dev(r), dev(off), dev(ids))
        e.check_errors()
        cnt = cnt.cpu().numpy()
        for b in range(37):
            bounds = _rank_bounds(ref[b], lists[b])
            exact = O.filtered_ranks(ref[b], lists[b])
            for j in range(off[b], off[b + 1]):
                rk = 1 + cnt[j]
                lo, hi = bounds[int(ids[j])]
                assert lo <= rk <= hi, (model, s, b, int(ids[j]), rk, lo, hi, exact[int(ids[j])])


def test_filtered_ranks_planted_and_sharded():
    from paper_2503_02172_b200.sharded import answers_csr
    from planted import PlantedKG
    from test_oracle_planted import planted_queries
    from paper_2503_02172_b200.kgq import RANK_DIST, RANK_COUNT
    kg = PlantedKG(n_entity=200, n_relation=12, dim=32, depth=4, seed=7)
    t = synth.make_tables("gqe", kg.n, 12, 32, seed=1)
    t["entity"], t["relation"] = kg.E.copy(), kg.R.copy()
    full = Engine("gqe", kg.n, 12, 32, max_batch=16, max_k=8)
    full.load_tables(t)
    for s in ("1p", "2p", "2u", "up"):
        a, r = planted_queries(kg, s, 12, seed=3)
        lists = [sorted(kg.answers(s, list(a[b]), list(r[b]))) for b in range(len(a))]
        off, ids = answers_csr(lists)
        _, cnt = full.rank_answers(s, dev(a), dev(r), dev(off), dev(ids))
        assert np.all(cnt.cpu().numpy() == 0), s   # every true answer has filtered rank 1
        # the two-phase protocol over W virtual shards gives the same counts as one shard
        rand = [np.unique(np.r_[lst, np.random.default_rng(b).choice(kg.n, 3, replace=False)])
                for b, lst in enumerate(lists)]
        off2, ids2 = answers_csr(rand)
        _, c_full = full.rank_answers(s, dev(a), dev(r), dev(off2), dev(ids2))
        for W in (2, 3):
            shards = []
            for rank in range(W):
                e = Engine("gqe", kg.n, 12, 32, max_batch=16, max_k=8, world_size=W, rank=rank)
                e.load_tables(t)
                shards.append(e)
            dists = [e.rank_answers(s, dev(a), dev(r), dev(off2), dev(ids2), mode=RANK_DIST)[0] for e in shards]
            ad = torch.stack(dists).min(0).values            # the min-all-reduce
            cnts = [e.rank_answers(s, dev(a), dev(r), dev(off2), dev(ids2), mode=RANK_COUNT, ans_dist=ad.clone())[1]
                    for e in shards]
            assert torch.equal(torch.stack(cnts).sum(0), c_full), (s, W)   # the sum-all-reduce
            for e in shards:
                e.close()


@pytest.mark.parametrize("N,k,model,fused", [(5000, 10, "gqe", "auto"), (5000, 32, "gqe", "auto"),
                                             (40000, 16, "gqe", "auto"), (5000, 10, "betae", "off"),
                                             (3000, 32, "betae", "auto"), (5000, 10, "betae", "on"),
                                             (20000, 16, "betae", "on")])
def test_topk_heavy_ties(N, k, model, fused):
    """Q13/Q15 with massive exact ties: 7 distinct entity rows repeated over the table, so every
    query has ~N/7 entities at exactly its best distance (bit-identical: same row, same
    arithmetic).  The top-k must be those ties in ascending id order -- the filter buffer of
    the top-k kernel overflows and folds many times; N > 32k also takes the chunked path; BetaE
    with k <= 16 takes the fused per-stripe lists of the scorer epilogue."""
    d, R, B = 16, 4, 20   # BetaE: 20 query rows take the tensor-core scorer + block-minima top-k
    rng = np.random.default_rng(5)
    w = d if model == "gqe" else 2 * d
    pat = rng.uniform(-0.9, 1, (7, w)).astype(np.float32)
    which = rng.integers(0, 7, N)
    t = synth.make_tables(model, N, R, d, hidden=8, seed=3)
    t["entity"] = pat[which].copy()
    e = Engine(model, N, R, d, hidden=8, max_batch=B, max_k=32)
    e.set_fused_topk(fused)
    e.load_tables(t)
    m = O.Model(model, t, dim=d)
    a, r = synth.make_queries("1p", B, N, R, seed=4)
    td, ti = e.submit("1p", dev(a), dev(r), k)
    e.check_errors()
    ref = m.scores("1p", a, r)
    td, ti = td.cpu().numpy(), ti.cpu().numpy()
    for b in range(B):
        best = np.min(ref[b])
        ties = np.nonzero(ref[b] == best)[0]
        assert len(ties) >= k
        np.testing.assert_array_equal(ti[b], ties[:k], err_msg=f"row {b}: tied ids not ascending")
        assert np.all(td[b] == td[b][0])
    e.close()


@pytest.mark.parametrize("s", ["1p", "3in", "up", "pni", "2u", "ip"])
def test_fused_topk_matches_distance_block_path(s):
    """the BetaE tensor-core scorer keeps every row's k smallest (dist, id) per N
    stripe in its epilogue (no [B, N] distance block; k <= 16) and a warp merge of the stripe
    lists gives the top-k.  Checked against the oracle, and bit for bit against the same submit
    with shard_dist (distance block written, block-minima top-k), for k = 1, 10, 16 and a batch
    of 61 queries (ragged 256-row blocks; fused forced ON, so the planner cuts the 1000-entity
    table into many stripes: up to 2 x 8 lists per row)."""
    e, m, t = engine("betae", max_batch=64)
    e.set_fused_topk("on")
    a, r = synth.make_queries(s, 61, SMALL["N"], SMALL["R"], seed=synth.query_seed(29, s))
    ref = m.scores(s, a, r)
    for k in (1, 10, 16):
        fd, fi = e.submit(s, dev(a), dev(r), k)
        bd, bi, _ = e.submit(s, dev(a), dev(r), k, shard_dist=True)
        e.check_errors()
        assert torch.equal(fi, bi), (s, k)
        assert torch.equal(fd, bd), (s, k)
        fd, fi = fd.cpu().numpy(), fi.cpu().numpy()
        for b in range(61):
            assert_topk_ok(fd[b], fi[b], ref[b], k, what=f"fused {s} k={k} row {b}")
    e.set_fused_topk("auto")


def test_fused_topk_many_stripes_and_option():
    """A 20,000-entity table with fused top-k forced ON: the planner cuts up to 64 stripes (128
    lists per row, four list heads per lane in the merge).  Bit-identical to the same context with
    the option OFF (distance block + block-minima top-k), through eager, captured and replayed
    submits (set_option re-captures the graphs), and checked against the oracle."""
    N, R, d = 20000, 10, 24
    t = synth.make_tables("betae", N, R, d, hidden=40, seed=12)
    m = O.Model("betae", t, dim=d)
    e = Engine("betae", N, R, d, hidden=40, max_batch=64, max_k=16)
    e.load_tables(t)
    for s in ("1p", "up"):
        a, r = synth.make_queries(s, 40, N, R, seed=77)
        outs = {}
        for mode in ("on", "off", "on"):
            e.set_fused_topk(mode)
            for _ in range(3):  # eager, capture, replay
                od, oi = e.submit(s, dev(a), dev(r), 16)
            outs.setdefault(mode, []).append((od.clone(), oi.clone()))
        e.check_errors()
        for od, oi in outs["on"]:
            assert torch.equal(oi, outs["off"][0][1]) and torch.equal(od, outs["off"][0][0]), s
        ref = m.scores(s, a, r)
        od, oi = outs["on"][0][0].cpu().numpy(), outs["on"][0][1].cpu().numpy()
        for b in range(40):
            assert_topk_ok(od[b], oi[b], ref[b], 16, what=f"many stripes {s} row {b}")
    from paper_2503_02172_b200 import kgq as K
    with pytest.raises(KgqError, match="EINVAL"):  # a value outside OFF / ON / AUTO
        e._check(K._lib.kgq_set_option(e._h, 1, 7))
    with pytest.raises(KgqError, match="EINVAL"):  # an unknown option
        e._check(K._lib.kgq_set_option(e._h, 99, 0))
    e.close()


def test_fused_topk_invalid_rows_and_tiny_table():
    """Fused top-k edge cases: a query with an out-of-range relation gets NaN / -1 (the other
    rows exact), and k = N on a 9-entity table (one ragged tile, most stripe lists padding)
    returns every entity in (distance, id) order."""
    e, m, t = engine("betae", max_batch=64)
    e.set_fused_topk("on")
    a, r = synth.make_queries("2p", 40, SMALL["N"], SMALL["R"], seed=3)
    r = r.copy()
    r[7, 1] = SMALL["R"] + 5
    td, ti = e.submit("2p", dev(a), dev(r), 12)
    with pytest.raises(KgqError, match="ERANGE"):
        e.check_errors()
    td, ti = td.cpu().numpy(), ti.cpu().numpy()
    assert np.all(np.isnan(td[7])) and np.all(ti[7] == -1)
    ok = [b for b in range(40) if b != 7]
    ref = m.scores("2p", a[ok], r[ok])
    for j, b in enumerate(ok):
        assert_topk_ok(td[b], ti[b], ref[j], 12)
    e.set_fused_topk("auto")
    N = 9
    t9 = synth.make_tables("betae", N, 5, 24, hidden=32, seed=4)
    e9 = Engine("betae", N, 5, 24, hidden=32, max_batch=32, max_k=16)
    e9.set_fused_topk("on")
    e9.load_tables(t9)
    a9, r9 = synth.make_queries("up", 30, N, 5, seed=6)
    td, ti = e9.submit("up", dev(a9), dev(r9), N)
    e9.check_errors()
    td, ti = td.cpu().numpy(), ti.cpu().numpy()
    ref9 = O.Model("betae", t9, dim=24).scores("up", a9, r9)
    for b in range(30):
        assert_topk_ok(td[b], ti[b], ref9[b], N, what=f"k = N row {b}")
        assert sorted(ti[b].tolist()) == list(range(N))
    e9.close()


def test_betae_out_of_range_relation_at_later_hop():
    """The first projection layer range-checks relation ids in its GEMM epilogue (relation
    term factored out): a bad hop-1 relation must still give KGQ_ERANGE and a
    NaN / -1 row, leaving the other rows exact."""
    e, m, t = engine("betae")
    a, r = synth.make_queries("3p", 20, SMALL["N"], SMALL["R"], seed=17)
    bad = r.copy()
    bad[3, 1] = SMALL["R"]
    bad[7, 2] = -5
    td, ti = e.submit("3p", dev(a), dev(bad), 5)
    with pytest.raises(KgqError, match="ERANGE"):
        e.check_errors()
    e.check_errors()
    td, ti = td.cpu().numpy(), ti.cpu().numpy()
    assert np.all(np.isnan(td[[3, 7]])) and np.all(ti[[3, 7]] == -1)
    ok = [b for b in range(20) if b not in (3, 7)]
    ref = m.scores("3p", a[ok], r[ok])
    for j, b in enumerate(ok):
        assert_topk_ok(td[b], ti[b], ref[j], 5)


@pytest.mark.parametrize("model,fused", [("betae", "auto"), ("betae", "on"), ("gqe", "auto")])
def test_mixed_structure_batch(model, fused):
    """kgq_submit_mixed: several structures in one call.  BetaE runs them
    level-synchronously (hops of all groups batched into one MLP, one scorer, one top-k), GQE
    group by group; every group's rows must match the oracle like a plain submit."""
    e, m, t = engine(model, max_batch=256)
    e.set_fused_topk(fused)
    N, R = SMALL["N"], SMALL["R"]
    structs = STRUCTS[model]
    groups, refs = [], []
    for i, s in enumerate(structs):
        B = 5 + (i * 7) % 11   # ragged group sizes
        a, r = synth.make_queries(s, B, N, R, seed=100 + i)
        groups.append((s, dev(a.astype(np.int32)), dev(r.astype(np.int32))))
        refs.append(m.scores(s, a, r))
    td, ti = e.submit_mixed(groups, 10)
    e.check_errors()
    td, ti = td.cpu().numpy(), ti.cpu().numpy()
    q = 0
    for (s, a, _), ref in zip(groups, refs):
        for b in range(a.shape[0]):
            assert_topk_ok(td[q + b], ti[q + b], ref[b], 10, what=f"mixed {model} {s} row {b}")
        q += a.shape[0]
    assert q == td.shape[0]
    e.set_fused_topk("auto")


def test_mixed_batch_aligned_groups_remap():
    """Groups of 32 / 64 queries: every hop segment is whole 32-row boxes, so the last MLP layer
    of each batched hop writes its rows straight into the state through the epilogue's row remap
    (no scatter kernel).  Every row against the oracle, both fused-top-k modes, and a bad relation
    id at a later hop still flags exactly its query."""
    e, m, t = engine("betae", max_batch=1024)
    N, R = SMALL["N"], SMALL["R"]
    structs = synth.ALL_STRUCTURES
    for fused in ("auto", "on"):
        e.set_fused_topk(fused)
        groups, refs = [], []
        for i, s in enumerate(structs):
            B = 32 if i % 2 else 64
            a, r = synth.make_queries(s, B, N, R, seed=900 + i)
            if s == "3p":
                r = r.copy()
                r[5, 2] = R + 1  # bad id at hop 2
            groups.append((s, dev(a.astype(np.int32)), dev(r.astype(np.int32))))
            refs.append((a, r))
        td, ti = e.submit_mixed(groups, 10)
        with pytest.raises(KgqError, match="ERANGE"):
            e.check_errors()
        td, ti = td.cpu().numpy(), ti.cpu().numpy()
        q = 0
        for (s, a, _), (qa, qr) in zip(groups, refs):
            B = a.shape[0]
            ok = [b for b in range(B) if not (s == "3p" and b == 5)]
            ref = m.scores(s, qa[ok], qr[ok])
            for j, b in enumerate(ok):
                assert_topk_ok(td[q + b], ti[q + b], ref[j], 10, what=f"aligned mixed {fused} {s} row {b}")
            if s == "3p":
                assert np.all(np.isnan(td[q + 5])) and np.all(ti[q + 5] == -1)
            q += B
    e.set_fused_topk("auto")


def test_mixed_batch_out_of_range_and_equivalence():
    """A bad relation id in one group flags exactly that query (global index); the other rows
    agree with one kgq_submit per group (same arithmetic, different batching: 1e-5)."""
    e, m, t = engine("betae", max_batch=256)
    N, R = SMALL["N"], SMALL["R"]
    groups = []
    for i, s in enumerate(("3p", "2u", "ip", "pni", "up-DM")):
        a, r = synth.make_queries(s, 12, N, R, seed=200 + i)
        if s == "ip":
            r = r.copy()
            r[4, 2] = R + 3   # post-intersection hop relation out of range
        groups.append((s, dev(a.astype(np.int32)), dev(r.astype(np.int32))))
    td, ti = e.submit_mixed(groups, 8)
    with pytest.raises(KgqError, match="ERANGE"):
        e.check_errors()
    e.check_errors()
    td, ti = td.cpu().numpy(), ti.cpu().numpy()
    bad = 2 * 12 + 4
    assert np.all(np.isnan(td[bad])) and np.all(ti[bad] == -1)
    q = 0
    for s, a, r in groups:
        sd, si = e.submit(s, a, r, 8)
        sd, si = sd.cpu().numpy(), si.cpu().numpy()
        for b in range(12):
            if q + b == bad:
                continue
            np.testing.assert_allclose(td[q + b], sd[b], rtol=1e-5, err_msg=f"{s} row {b}")
        q += 12
    with pytest.raises(KgqError, match="ERANGE"):  # the per-group "ip" submit re-flags the bad id
        e.check_errors()


def test_virtual_shards_mixed_batch():
    """kgq_submit_mixed on W entity shards + kgq_merge_topk == one shard, bit for bit."""
    N, R, d = 1000, 20, 40
    t = synth.make_tables("betae", N, R, d, hidden=96, seed=5)
    groups = []
    for i, s in enumerate(("2p", "up", "3in", "ip", "2u-DM")):
        a, r = synth.make_queries(s, 9 + i, N, R, seed=40 + i)
        groups.append((s, dev(a.astype(np.int32)), dev(r.astype(np.int32))))
    full = Engine("betae", N, R, d, hidden=96, max_batch=128, max_k=32)
    full.load_tables(t)
    fd, fi = full.submit_mixed(groups, 12)
    m = O.Model("betae", t, dim=d)
    refs = [m.scores(s, a.cpu().numpy(), r.cpu().numpy()) for s, a, r in groups]
    for W in (2, 3):
        parts = []
        for rank in range(W):
            e = Engine("betae", N, R, d, hidden=96, max_batch=128, max_k=32, world_size=W, rank=rank)
            e.load_tables(t)
            parts.append(e.submit_mixed(groups, 12))
            torch.cuda.synchronize()
            e.close()
        md, mi = full.merge_topk(torch.stack([p[0] for p in parts]), torch.stack([p[1] for p in parts]), 12)
        mdn, min_ = md.cpu().numpy(), mi.cpu().numpy()
        q = 0
        for (s, a, _), ref in zip(groups, refs):
            for b in range(a.shape[0]):
                assert_topk_ok(mdn[q + b], min_[q + b], ref[b], 12, what=f"merged mixed W={W} {s} row {b}")
            q += a.shape[0]
        assert torch.equal(mi, fi), W
        assert torch.equal(md, fd), W
    full.close()


@pytest.mark.parametrize("model", ["betae", "gqe"])
def test_scorer_row_chunks(model):
    """Batches larger than the distance scratch are scored in chunks of rows (kgq_api.cu bchunk:
    each chunk re-reads the table).  KGQ_DIST_BUDGET_MB = 7 on a 100K-entity table gives 18-query
    chunks, so B = 37 runs two tensor-core / tiled chunks and a 1-query streaming chunk (BetaE), and
    a mixed submit larger than one chunk falls back to group-by-group submits.  Every row vs the
    oracle (top-k ids and distances, tie-aware)."""
    import os
    N, R, d, H, B, k = 100_003, 20, 16, 32, 37, 10
    t = synth.make_tables(model, N, R, d, hidden=H, seed=31)
    os.environ["KGQ_DIST_BUDGET_MB"] = "7"
    try:
        e = Engine(model, N, R, d, hidden=H, max_batch=128, max_k=k)
        e.load_tables(t)  # the scratch is sized at finalize
    finally:
        del os.environ["KGQ_DIST_BUDGET_MB"]
    m = O.Model(model, t, dim=d)
    groups, refs = [], []
    for s in ("1p", "2u", "ip"):
        a, r = synth.make_queries(s, B, N, R, seed=synth.query_seed(31, s))
        td, ti = e.submit(s, dev(a), dev(r), k)
        e.check_errors()
        ref = m.scores(s, a, r)
        td, ti = td.cpu().numpy(), ti.cpu().numpy()
        for b in range(B):
            assert_topk_ok(td[b], ti[b], ref[b], k, what=f"chunked {model} {s} row {b}")
        groups.append((s, dev(a.astype(np.int32)), dev(r.astype(np.int32))))
        refs.append(ref)
    md, mi = e.submit_mixed(groups, k)
    e.check_errors()
    md, mi = md.cpu().numpy(), mi.cpu().numpy()
    for gi, ref in enumerate(refs):
        for b in range(B):
            assert_topk_ok(md[gi * B + b], mi[gi * B + b], ref[b], k, what=f"chunked mixed {model} row {b}")
    e.close()


def test_streaming_scorer_shared_memory_limit_across_dims():
    """The small-batch streaming scorers stage the query rows in dynamic shared memory sized
    d x rows: a d = 40 context first (5 KB for BetaE 2u at B = 8), then a d = 400 one in the same
    process (51 KB, above the 48 KB default) -- the opt-in limit is cached per call site and must
    only ever be raised (a cached "done" flag once left it at 5 KB: invalid argument)."""
    for d, N in ((40, 1000), (400, 3000)):
        t = synth.make_tables("betae", N, 20, d, hidden=64, seed=41)
        e = Engine("betae", N, 20, d, hidden=64, max_batch=8, max_k=10)
        e.load_tables(t)
        m = O.Model("betae", t, dim=d)
        a, r = synth.make_queries("2u", 8, N, 20, seed=42)
        td, ti = e.submit("2u", dev(a), dev(r), 10)
        e.check_errors()
        ref = m.scores("2u", a, r)
        td, ti = td.cpu().numpy(), ti.cpu().numpy()
        for b in range(8):
            assert_topk_ok(td[b], ti[b], ref[b], 10, what=f"stream d={d} row {b}")
        e.close()


def test_mixed_graph_replay_matches_eager():
    """The second identical kgq_submit_mixed is captured into a CUDA graph and later calls
    replay it (inputs repacked into the same staging buffers, new query content every round):
    bit-identical to an engine that runs every call eagerly (KGQ_NO_GRAPHS=1)."""
    import os
    N, R, d, H = 1000, 20, 40, 96
    t = synth.make_tables("betae", N, R, d, hidden=H, seed=5)
    eg = Engine("betae", N, R, d, hidden=H, max_batch=128, max_k=16)
    eg.load_tables(t)
    os.environ["KGQ_NO_GRAPHS"] = "1"
    try:
        ee = Engine("betae", N, R, d, hidden=H, max_batch=128, max_k=16)
    finally:
        del os.environ["KGQ_NO_GRAPHS"]
    ee.load_tables(t)
    shapes = [("2p", 9), ("up", 11), ("3in", 7), ("ip", 5), ("2u-DM", 6)]
    Q = sum(b for _, b in shapes)
    out = (torch.empty((Q, 12), device="cuda"), torch.empty((Q, 12), dtype=torch.int32, device="cuda"))
    for rnd in range(4):
        groups = []
        for i, (s, b) in enumerate(shapes):
            a, r = synth.make_queries(s, b, N, R, seed=300 + 10 * rnd + i)
            groups.append((s, dev(a.astype(np.int32)), dev(r.astype(np.int32))))
        gd, gi = eg.submit_mixed(groups, 12, out=out)
        ed, ei = ee.submit_mixed(groups, 12)
        torch.cuda.synchronize()
        assert torch.equal(gi, ei), rnd
        assert torch.equal(gd, ed), rnd
    eg.check_errors()
    ee.check_errors()
    eg.close()
    ee.close()


def test_mixed_host_submit_matches_device_and_oracle():
    """kgq_submit_mixed_host_async (bench.py's end-to-end call): pinned host inputs packed in
    group order, host outputs.  Every row checked against the oracle, and bit-identical to the
    device-pointer mixed submit over rounds that go eager -> capture -> graph replay, with new
    query content every round (the staging buffers' addresses are what the graph keys on)."""
    N, R, d, H = 1000, 20, 40, 96
    t = synth.make_tables("betae", N, R, d, hidden=H, seed=8)
    m = O.Model("betae", t, dim=d)
    eh = Engine("betae", N, R, d, hidden=H, max_batch=160, max_k=16)
    eh.load_tables(t)
    ed = Engine("betae", N, R, d, hidden=H, max_batch=160, max_k=16)
    ed.load_tables(t)
    shapes = [("3i", 13), ("up", 9), ("pni", 17), ("1p", 6), ("inp", 11), ("2u-DM", 5)]
    ss, bs = [s for s, _ in shapes], [b for _, b in shapes]
    Q = sum(bs)
    k = 12
    hd = torch.empty((Q, k)).pin_memory()
    hi = torch.empty((Q, k), dtype=torch.int32).pin_memory()
    st = torch.cuda.Stream()
    for rnd in range(4):
        qs = [synth.make_queries(s, b, N, R, seed=700 + 10 * rnd + i) for i, (s, b) in enumerate(shapes)]
        a = torch.from_numpy(np.concatenate([x[0].reshape(-1) for x in qs]).astype(np.int32)).pin_memory()
        r = torch.from_numpy(np.concatenate([x[1].reshape(-1) for x in qs]).astype(np.int32)).pin_memory()
        eh.submit_mixed_host(ss, bs, a.numpy(), r.numpy(), k, (hd.numpy(), hi.numpy()), stream=st)
        st.synchronize()
        dd, di = ed.submit_mixed([(s, dev(x[0].astype(np.int32)), dev(x[1].astype(np.int32)))
                                  for s, x in zip(ss, qs)], k)
        torch.cuda.synchronize()
        assert np.array_equal(hi.numpy(), di.cpu().numpy()), rnd
        assert np.array_equal(hd.numpy(), dd.cpu().numpy()), rnd
        if rnd in (0, 3):
            q = 0
            for (s, b), (qa, qr) in zip(shapes, qs):
                ref = m.scores(s, qa, qr)
                for j in range(b):
                    assert_topk_ok(hd.numpy()[q + j], hi.numpy()[q + j], ref[j], k, what=f"host mixed {s} row {j}")
                q += b
    eh.check_errors()
    ed.check_errors()
    with pytest.raises(KgqError, match="EINVAL"):  # more queries than max_batch
        eh.submit_mixed_host(["1p"], [161], np.zeros(161, np.int32), np.zeros(161, np.int32), k,
                             (np.empty((161, k), np.float32), np.empty((161, k), np.int32)))
    eh.close()
    ed.close()


def test_ktime_launch_spans():
    """kgq_ktime_*: every tcgen05 GEMM launch of a submit logs one in-kernel span (bench.py's
    roofline time); the per-stage sums equal the logged spans, and toggling keeps results
    bit-identical (the graphs are re-captured with the accounting pointer)."""
    e, m, t = engine("betae")
    a, r = synth.make_queries("up", 20, SMALL["N"], SMALL["R"], seed=2)
    ref_d, ref_i = e.submit("up", dev(a), dev(r), 5)
    e.ktime(True)
    e.ktime_read()
    e.ktime_log()
    for _ in range(3):  # eager, capture, replay
        d_, i_ = e.submit("up", dev(a), dev(r), 5)
        assert torch.equal(i_, ref_i) and torch.equal(d_, ref_d)
    kt = e.ktime_read()
    log = e.ktime_log()
    e.ktime(False)
    n_dense, n_score = kt["dense"][1], kt["score"][1]
    assert n_dense > 0 and n_score == 3          # up: one scorer GEMM per submit
    assert len(log) == n_dense + n_score
    assert np.all(log[:, 1] > log[:, 0])
    for st, name in ((0, "dense"), (1, "score")):
        sel = log[log[:, 2] == st]
        np.testing.assert_allclose((sel[:, 1] - sel[:, 0]).sum() * 1e-6, kt[name][0], rtol=1e-9)


def test_concurrent_contexts_on_streams_match_sequential():
    """bench.py's headline form: the per-type submits dealt over three streams, one context per
    stream, overlapping on the GPU -- every result bit-identical to one context on one stream,
    and checked against the oracle (the contexts share no scratch)."""
    N, R, d, H = 1000, 20, 40, 96
    t = synth.make_tables("betae", N, R, d, hidden=H, seed=31)
    m = O.Model("betae", t, dim=d)
    engs = []
    for _ in range(3):
        e = Engine("betae", N, R, d, hidden=H, max_batch=64, max_k=16)
        e.load_tables(t)
        engs.append(e)
    structs = synth.ALL_STRUCTURES
    qs = {s: synth.make_queries(s, 40, N, R, seed=500 + i) for i, s in enumerate(structs)}
    dq = {s: (dev(a), dev(r)) for s, (a, r) in qs.items()}
    seq = {s: engs[0].submit(s, *dq[s], 10) for s in structs}
    torch.cuda.synchronize()
    seq = {s: (x[0].clone(), x[1].clone()) for s, x in seq.items()}
    streams = [torch.cuda.Stream() for _ in range(3)]
    for rnd in range(3):  # eager, capture, replay
        outs = {}
        for i, s in enumerate(structs):
            j = i % 3
            outs[s] = engs[j].submit(s, *dq[s], 10, stream=streams[j])
        torch.cuda.synchronize()
        for s in structs:
            assert torch.equal(outs[s][1], seq[s][1]) and torch.equal(outs[s][0], seq[s][0]), (rnd, s)
    for s in ("2u", "pni", "up-DM"):
        a, r = qs[s]
        ref = m.scores(s, a, r)
        gd, gi = outs[s][0].cpu().numpy(), outs[s][1].cpu().numpy()
        for b in range(40):
            assert_topk_ok(gd[b], gi[b], ref[b], 10, what=f"concurrent {s} row {b}")
    for e in engs:
        e.check_errors()
        e.close()
