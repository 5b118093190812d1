"""Pins for the N1 filtered-ranking oracle (-m "not gpu")."""
import numpy as np
import pytest

import oracle as O


def test_mrr_examples_from_spec():
    # answer ranked 1 -> 1.0; answer ranked 4 -> 0.25
    assert O.mrr_hits([1])[0] == 1.0
    assert O.mrr_hits([4])[0] == 0.25
    assert O.mrr_hits([1, 4]) == (0.625, 0.5, 0.5, 1.0)


def test_filtered_rank_against_explicit_sort():
    rng = np.random.default_rng(0)
    for trial in range(20):
        n = 60
        d = rng.integers(0, 15, size=n).astype(np.float64)   # many ties
        ans = rng.choice(n, size=rng.integers(1, 8), replace=False)
        fr = O.filtered_ranks(d, ans)
        order = sorted(range(n), key=lambda e: (d[e], e))      # full sort, ties by id
        for a in ans:
            pos = order.index(a)                               # 0-based raw rank
            n_ans_before = sum(1 for e in order[:pos] if e in set(ans))
            assert fr[int(a)] == pos - n_ans_before + 1        # KGReasoning: rank - #answers before + 1


def test_filtered_rank_ignores_other_answers_and_shards_add_up():
    d = np.array([0.5, 0.1, 0.3, 0.2, 0.9])
    # answers {1, 3}: entity 1 first (rank 1); entity 3 is behind 1 (an answer, filtered) -> rank 1
    assert O.filtered_ranks(d, [1, 3]) == {1: 1, 3: 1}
    # answer {0}: non-answers 1, 2, 3 are closer -> rank 4
    assert O.filtered_ranks(d, [0]) == {0: 4}
    # sharded counting: rank = 1 + sum over shards of #better non-answers in the shard
    rng = np.random.default_rng(1)
    d = rng.random(101)
    ans = [3, 50, 99]
    full = O.filtered_ranks(d, ans)
    for W in (2, 3):
        tot = {a: 1 for a in ans}
        for r in range(W):
            lo, hi = O.shard_range(101, W, r)
            for a in ans:
                better = [(d[e] < d[a]) or (d[e] == d[a] and e < a) for e in range(lo, hi) if e not in ans]
                tot[a] += sum(better)
        assert tot == full
