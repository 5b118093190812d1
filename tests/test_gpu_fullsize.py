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
        _, _, sd = e.submit(s, dev(a), dev(r), 10, shard_dist=True)
        assert_dist_close(sd[torch.from_numpy(rows).cuda()].cpu().numpy(), ref, what=f"{name} {s} full rows")
        qe = e.query_embedding(s, dev(a), dev(r)).cpu().numpy()[rows]
        ref_q = m.query_embedding(s, a[rows], r[rows])
        # chain at H = 1600: the same per-structure bounds as the small configs
        assert_embedding_close(qe, ref_q, rel=chain_tolerance(s, "kgr-init", model), what=f"{name} {s} chain")


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
