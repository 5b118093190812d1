"""Whole-path brute force for the oracle on a planted integer KG (GQE).

The symbolic set-semantics answer (tests/planted.py) must be exactly the set of
entities the oracle ranks at distance 0, for 1p/2p/3p/2i/3i/2u/up queries drawn
answers-first.  Pins plan slot order (which relation goes with which hop), the
union-as-min reading and the top-k (dist, id) order end to end.
"""
import numpy as np
import pytest

import oracle as O
from planted import PlantedKG

import synth


def gqe_model(kg):
    t = synth.make_tables("gqe", kg.n, kg.R.shape[0], kg.E.shape[1], seed=1)
    t["entity"] = kg.E.copy()
    t["relation"] = kg.R.copy()
    return O.Model("gqe", t, dim=kg.E.shape[1])


def planted_queries(kg, structure, n, seed):
    rng = np.random.default_rng(seed)
    A, R = [], []
    for _ in range(n):
        if structure in ("1p", "2p", "3p"):
            L = int(structure[0])
            a, rels, _ = kg.sample_chain(rng, L)
            A.append([a]); R.append(rels)
        elif structure in ("2i", "3i"):
            a, rels, t = kg.sample_chain(rng, 1)
            k = int(structure[0])
            A.append([a] * k); R.append(rels * k)
        elif structure == "2u":
            a0, r0, _ = kg.sample_chain(rng, 1)
            a1, r1, _ = kg.sample_chain(rng, 1)
            A.append([a0, a1]); R.append([r0[0], r1[0]])
        elif structure == "up":
            a0, r0, _ = kg.sample_chain(rng, 2)
            # second clause ends with the same last relation slot (shared r2)
            cands = [(h, r, t) for (h, r, t) in kg.triples if (t, r0[1]) in kg.adj]
            h, r, _ = cands[rng.integers(0, len(cands))]
            A.append([a0, h]); R.append([r0[0], r, r0[1]])
    return np.array(A, np.int32), np.array(R, np.int32)


@pytest.mark.parametrize("structure", ["1p", "2p", "3p", "2i", "3i", "2u", "up"])
def test_planted_answers_are_the_zero_distance_set(structure):
    kg = PlantedKG(n_entity=200, n_relation=12, dim=32, depth=4, seed=7)
    m = gqe_model(kg)
    a, r = planted_queries(kg, structure, 12, seed=hash(structure) % 1000)
    dist = m.scores(structure, a, r)
    td, ti = O.topk(dist, 4)
    for b in range(len(a)):
        ans = kg.answers(structure, list(a[b]), list(r[b]))
        assert ans, "answers-first sampling must give a non-empty answer set"
        zero = set(np.nonzero(dist[b] <= 1e-9)[0].tolist())
        assert zero == ans
        # top-k order: the answers first, by ascending id, then positive distances
        n = len(ans)
        assert list(ti[b, :n]) == sorted(ans)
        assert td[b, n] > 0.5
