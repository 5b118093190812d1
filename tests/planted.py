"""Planted integer knowledge graph + set-semantics answer oracle (test helper).

SPEC S:58-66 (answer_oracle): projection = union of neighbours over the frontier,
intersection = set intersection, union = set union.  The planted KG is a forest in
which every edge (h, r, t) satisfies E[t] = E[h] + R[r] exactly with small integers, so
GQE (translation projection) puts each answer at L1 distance exactly 0 in fp32 and in
float64 alike.  Construction rules that make answers unique:
  * relations are partitioned by depth (a node at depth k only uses relations of group k),
    so the relation multiset of a path determines its order;
  * a parent never uses the same relation twice, so (node, relation path) has <= 1 endpoint;
  * relation vectors and root vectors are random integers drawn so that distinct
    (root, relation multiset) sums differ (checked: all embeddings are distinct).
"""
from __future__ import annotations

import numpy as np


class PlantedKG:
    def __init__(self, n_entity=200, n_relation=12, dim=32, depth=4, seed=7, n_roots=3):
        rng = np.random.default_rng(seed)
        assert n_relation % depth == 0
        per = n_relation // depth
        self.R = rng.integers(-40, 41, size=(n_relation, dim)).astype(np.float32)
        self.E = np.zeros((n_entity, dim), np.float32)
        self.E[:n_roots] = rng.integers(-2000, 2001, size=(n_roots, dim)).astype(np.float32)
        self.depth_of = np.zeros(n_entity, np.int64)
        self.adj: dict[tuple[int, int], set[int]] = {}
        used: dict[int, set[int]] = {}
        self.triples = []
        t = n_roots
        frontier = list(range(n_roots))
        while t < n_entity:
            cand = [h for h in frontier if self.depth_of[h] < depth
                    and len(used.get(h, ())) < per]
            if not cand:
                break
            h = int(cand[rng.integers(0, len(cand))])
            k = int(self.depth_of[h])
            free = [r for r in range(k * per, (k + 1) * per) if r not in used.get(h, set())]
            r = int(free[rng.integers(0, len(free))])
            used.setdefault(h, set()).add(r)
            self.E[t] = self.E[h] + self.R[r]
            self.depth_of[t] = k + 1
            self.adj.setdefault((h, r), set()).add(t)
            self.triples.append((h, r, t))
            frontier.append(t)
            t += 1
        self.n = t
        self.E = self.E[:t]
        # all embeddings distinct -> distance 0 identifies the entity uniquely
        assert len({row.tobytes() for row in self.E}) == self.n

    # -- set semantics ------------------------------------------------------
    def proj(self, frontier, r):
        out = set()
        for h in frontier:
            out |= self.adj.get((h, r), set())
        return out

    def answers(self, structure, anchors, rels):
        a = anchors
        r = rels
        p = self.proj
        if structure == "1p":
            return p({a[0]}, r[0])
        if structure == "2p":
            return p(p({a[0]}, r[0]), r[1])
        if structure == "3p":
            return p(p(p({a[0]}, r[0]), r[1]), r[2])
        if structure == "2i":
            return p({a[0]}, r[0]) & p({a[1]}, r[1])
        if structure == "3i":
            return p({a[0]}, r[0]) & p({a[1]}, r[1]) & p({a[2]}, r[2])
        if structure == "2u":
            return p({a[0]}, r[0]) | p({a[1]}, r[1])
        if structure == "up":
            return p(p({a[0]}, r[0]), r[2]) | p(p({a[1]}, r[1]), r[2])
        raise NotImplementedError(structure)

    def sample_chain(self, rng, length):
        """Answers-first: pick a target at depth >= length, walk back `length` edges."""
        parent = {t: (h, r) for (h, r, t) in self.triples}
        cands = [t for t in range(self.n) if self.depth_of[t] >= length]
        t = int(cands[rng.integers(0, len(cands))])
        rels = []
        node = t
        for _ in range(length):
            h, r = parent[node]
            rels.append(r)
            node = h
        return node, rels[::-1], t
