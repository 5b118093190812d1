"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times:
the whole batch runs on the GPU; the oracle checks a sample of queries (full distance rows
where it can afford them, sampled entities for the 2M-entity table)."""
import numpy as np
import pytest

import oracle as O
import synth
from parity import (assert_dist_close, assert_embedding_close, assert_topk_ok, assert_topk_ok_sampled,
                    chain_tolerance)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)
from paper_2503_02172_b200 import Engine  # noqa: E402

# (name, model, N, R, d, H, B, structures) -- BASELINE.json configs[1..3]
CONFIGS = [
    ("betae_fb15k237", "betae", 14505, 237, 400, 1600, 1024, synth.ALL_STRUCTURES),
    ("q2b_nell995", "q2b", 63361, 200, 400, 1600, 1024, synth.EPFO),
    ("betae_fb15k_neg", "betae", 14951, 1345, 400, 1600, 4096, synth.NEGATION),
]


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("cfg", CONFIGS, ids=[c[0] for c in CONFIGS])
def test_full_size_sampled(cfg):
    name, model, N, R, d, H, B, structs = cfg
    seed = 2503_02172 + [c[0] for c in CONFIGS].index(name) + 1
    t = synth.make_tables(model, N, R, d, hidden=H, seed=seed)
    e = Engine(model, N, R, d, hidden=H, max_batch=B, max_k=16)
    e.load_tables(t)
    m = O.Model(model, t, dim=d)
    rng = np.random.default_rng(0)
    for s in structs:
        a, r = synth.make_queries(s, B, N, R, seed=synth.query_seed(seed, s))
        td, ti = e.submit(s, dev(a), dev(r), 10)
        e.check_errors()
        td, ti = td.cpu().numpy(), ti.cpu().numpy()
        assert np.all(np.isfinite(td))
        # sampled rows include the first and the ragged last one
        rows = np.unique(np.r_[0, rng.integers(0, B, size=1), B - 1])
        ref = m.scores(s, a[rows], r[rows])
        for j, b in enumerate(rows):
            assert_topk_ok(td[b], ti[b], ref[j], 10, what=f"{name} {s} row {b}")
        # whole distance rows at the real K = 800 contraction (north_star: 1e-4 relative)
        bd, bi, sd = e.submit(s, dev(a), dev(r), 10, shard_dist=True)
        assert_dist_close(sd[torch.from_numpy(rows).cuda()].cpu().numpy(), ref, what=f"{name} {s} full rows")
        # BetaE: the first submit took the fused top-k (per-stripe lists in the scorer epilogue,
        # no distance block), this one the distance block + block-minima top-k: same values, so
        # the whole batch's top-k must agree bit for bit
        np.testing.assert_array_equal(bi.cpu().numpy(), ti, err_msg=f"{name} {s} fused vs block top-k ids")
        np.testing.assert_array_equal(bd.cpu().numpy(), td, err_msg=f"{name} {s} fused vs block top-k dists")
        qe = e.query_embedding(s, dev(a), dev(r)).cpu().numpy()[rows]
        ref_q = m.query_embedding(s, a[rows], r[rows])
        # chain at H = 1600: the same per-structure bounds as the small configs
        assert_embedding_close(qe, ref_q, rel=chain_tolerance(s, "kgr-init", model), what=f"{name} {s} chain")


def test_full_size_mixed_step_as_benched():
    """bench.py's headline step: ONE kgq_submit_mixed of all 14 BetaE types x 1024 queries at the
    FB15k-237 shape (the same tables, queries and launch configuration the bench times; the
    scorer launch of the 12,288 single-branch rows takes the fused top-k under AUTO).  Sampled rows
    of every type against the oracle (tie-aware top-k), and the whole batch bit for bit against
    the same submit with the fused top-k OFF (distance block + block-minima top-k)."""
    N, R, d, H, B = 14505, 237, 400, 1600, 1024
    seed = 2503_02172 + 1
    t = synth.make_tables("betae", N, R, d, hidden=H, seed=seed)
    e = Engine("betae", N, R, d, hidden=H, max_batch=14 * B, max_k=16)
    e.load_tables(t)
    m = O.Model("betae", t, dim=d)
    qs = [synth.make_queries(s, B, N, R, seed=synth.query_seed(seed, s)) for s in synth.STRUCTURES]
    a = dev(np.concatenate([q[0].reshape(-1) for q in qs]).astype(np.int32))
    r = dev(np.concatenate([q[1].reshape(-1) for q in qs]).astype(np.int32))
    out = (torch.empty((14 * B, 10), device="cuda"), torch.empty((14 * B, 10), dtype=torch.int32, device="cuda"))
    res = {}
    for mode in ("auto", "off"):
        e.set_fused_topk(mode)
        for _ in range(3):  # eager, capture, replay (the bench times replays)
            e.submit_mixed_packed(list(synth.STRUCTURES), [B] * 14, a, r, 10, out)
        e.check_errors()
        res[mode] = (out[0].cpu().numpy().copy(), out[1].cpu().numpy().copy())
    np.testing.assert_array_equal(res["auto"][1], res["off"][1])
    np.testing.assert_array_equal(res["auto"][0], res["off"][0])
    td, ti = res["auto"]
    assert np.all(np.isfinite(td))
    rng = np.random.default_rng(3)
    for i, s in enumerate(synth.STRUCTURES):
        rows = np.unique(np.r_[0, rng.integers(0, B), B - 1])
        ref = m.scores(s, qs[i][0][rows], qs[i][1][rows])
        for j, b in enumerate(rows):
            assert_topk_ok(td[i * B + b], ti[i * B + b], ref[j], 10, what=f"mixed full-size {s} row {b}")
    e.close()


def test_2m_entity_table_gqe_and_betae():
    """BASELINE.json configs[4] (1 shard): GQE and BetaE scoring over 2M entities, d 400.
    GQE: full oracle rows for 2 queries; BetaE: returned ids + a 20k-entity sample."""
    N, R, d = 2_000_000, 200, 400
    rng = np.random.default_rng(1)
    for model in ("gqe", "betae"):
        t = synth.make_tables(model, N, R, d, hidden=1600, seed=77)
        e = Engine(model, N, R, d, hidden=1600, max_batch=8, max_k=16)
        e.load_tables(t)
        m = O.Model(model, t, dim=d)
        a, r = synth.make_queries("1p", 8, N, R, seed=3)
        td, ti = e.submit("1p", dev(a), dev(r), 10)
        e.check_errors()
        td, ti = td.cpu().numpy(), ti.cpu().numpy()
        for b in (0, 7):
            q = m.query_embedding("1p", a[b:b + 1], r[b:b + 1])[:, 0]
            if model == "gqe":
                row = np.concatenate([m.distance(q, m.entity_view(np.arange(c, min(N, c + 200_000))))[0]
                                      for c in range(0, N, 200_000)])
                assert_topk_ok(td[b], ti[b], row, 10, what=f"2M gqe row {b}")
            else:
                samp = rng.choice(N, 20_000, replace=False)
                ref_s = m.distance(q, m.entity_view(samp))[0]
                ref_ids = m.distance(q, m.entity_view(ti[b].astype(np.int64)))[0]
                assert_topk_ok_sampled(td[b], ti[b], ref_ids, samp, ref_s, 10, what=f"2M betae row {b}")
        e.close()
        del t
