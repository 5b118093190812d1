"""Float64 CPU oracle for the CLQA query-embedding inference hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product path (``paper_2503_02172_b200``) never imports it, and this
module never imports the product path; the two share no code.  Inputs come from
``synth`` (random draws only).

What it computes (readings §8(c) Q1-Q21):
plain, unfused definitions of the GQE / Query2Box / BetaE operators, evaluated
in float64 on the fp32 tables (promoted), then the distance to every entity, the
DNF-union min, and a full sort by (distance, entity id).

Citations: ``P:n`` = /root/reference/PAPER.md line n; ``S:n`` = SPEC.md line n;
[ext] = operator semantics of the KGReasoning framework that the paper compiles
"without requiring additional manual modifications" (P:7), recorded here as
named constants / flags so a reading can be changed in one place.

Parity status per function is stated in each docstring ("pinned by" = which
``-m "not gpu"`` test fixes it against something other than this file).
"""
from __future__ import annotations

import numpy as np
from scipy.special import digamma, gammaln

# ----------------------------------------------------------------------------------------
# Readings of the paper, one constant each.
# ----------------------------------------------------------------------------------------
#: Q9: logit = gamma - distance; the oracle returns distances.  [ext]
GAMMA = {"gqe": 24.0, "q2b": 24.0, "betae": 60.0}
#: Q10: Query2Box weight of the inside distance ("box_mode (none, 0.02)").  [ext]
Q2B_CEN = 0.02
#: Q2 / Q12: BetaE regulariser  x -> clamp(x + 1, 0.05, 1e9)  [ext], applied to entity
#: rows (anchors and scored entities) and as the projection terminal.
REG_ADD, REG_MIN, REG_MAX = 1.0, 0.05, 1e9
#: Q2 flag: literal Eq. 4 terminal (softmax over the 2d outputs) then max(., 1e-6)
#:.
SOFTMAX_FLOOR = 1e-6
TERMINAL_REGULARIZER = "regularizer"
TERMINAL_SOFTMAX = "softmax"

STRUCTURES = ("1p", "2p", "3p", "2i", "3i", "pi", "ip", "2u", "up",
              "2in", "3in", "inp", "pin", "pni", "2u-DM", "up-DM")

# ----------------------------------------------------------------------------------------
# Computation plans per structure (SURVEY §8(b) slot table; Fig. 1 names P:17; Eq. 1
# DNF; KGReasoning flattened slot order [ext]).  Node kinds:
#   ('A', i)          anchor slot i                        e_i -> var_i        (Eq. 2)
#   ('P', x, j)       projection of x by relation slot j   exists / r(e,v)     (Eq. 2)
#   ('I', [x...])     intersection                         and -> f_and        (Eq. 2)
#   ('N', x)          negation                             not -> f_not        (Eq. 2)
#   ('U', [x...])     union, top level only (DNF, Eq. 1)   or -> f_or          (Eq. 2)
# ----------------------------------------------------------------------------------------
A, P, I, N, U = "A", "P", "I", "N", "U"
PLANS = {
    "1p": (P, (A, 0), 0),
    "2p": (P, (P, (A, 0), 0), 1),
    "3p": (P, (P, (P, (A, 0), 0), 1), 2),
    "2i": (I, [(P, (A, 0), 0), (P, (A, 1), 1)]),
    "3i": (I, [(P, (A, 0), 0), (P, (A, 1), 1), (P, (A, 2), 2)]),
    "pi": (I, [(P, (P, (A, 0), 0), 1), (P, (A, 1), 2)]),
    "ip": (P, (I, [(P, (A, 0), 0), (P, (A, 1), 1)]), 2),
    "2u": (U, [(P, (A, 0), 0), (P, (A, 1), 1)]),
    "up": (U, [(P, (P, (A, 0), 0), 2), (P, (P, (A, 1), 1), 2)]),
    "2in": (I, [(P, (A, 0), 0), (N, (P, (A, 1), 1))]),
    "3in": (I, [(P, (A, 0), 0), (P, (A, 1), 1), (N, (P, (A, 2), 2))]),
    "inp": (P, (I, [(P, (A, 0), 0), (N, (P, (A, 1), 1))]), 2),
    "pin": (I, [(P, (P, (A, 0), 0), 1), (N, (P, (A, 1), 2))]),
    "pni": (I, [(N, (P, (P, (A, 0), 0), 1)), (P, (A, 1), 2)]),
    # De Morgan union, U(x, y) = N(I(N(x), N(y))) -- BetaE's alternative to
    # the DNF min (KGReasoning "2u-DM" / "up-DM" [ext]); one embedding, no top-level union.
    "2u-DM": (N, (I, [(N, (P, (A, 0), 0)), (N, (P, (A, 1), 1))])),
    "up-DM": (P, (N, (I, [(N, (P, (A, 0), 0)), (N, (P, (A, 1), 1))])), 2),
}


def _count(node, kind):
    k = node[0]
    if k == A:
        return 1 if kind == A else 0
    if k == P:
        return (1 if kind == P else 0) + _count(node[1], kind)
    if k == N:
        return _count(node[1], kind)
    return sum(_count(c, kind) for c in node[1])


def n_anchors(s):
    return _count(PLANS[s], A)


def n_relations(s):
    # distinct relation slots (up shares slot 2 between its two DNF clauses)
    slots = set()

    def walk(n):
        if n[0] == P:
            slots.add(n[2])
            walk(n[1])
        elif n[0] == N:
            walk(n[1])
        elif n[0] in (I, U):
            for c in n[1]:
                walk(c)
    walk(PLANS[s])
    return len(slots)


def n_branches(s):
    return len(PLANS[s][1]) if PLANS[s][0] == U else 1


def uses_negation(s):
    def walk(n):
        if n[0] == N:
            return True
        if n[0] == P:
            return walk(n[1])
        if n[0] in (I, U):
            return any(walk(c) for c in n[1])
        return False
    return walk(PLANS[s])


# ----------------------------------------------------------------------------------------
# Elementary pieces
# ----------------------------------------------------------------------------------------
def f64(x):
    return np.asarray(x, dtype=np.float64)


def linear(x, W, b):
    """torch.nn.Linear: y = x W^T + b, W is [out, in].  Pinned by test_oracle_ops
    (against torch.nn.functional.linear in float64 on a non-square W)."""
    return f64(x) @ f64(W).T + f64(b)


def relu(x):
    return np.maximum(x, 0.0)


def softmax(x, axis):
    m = np.max(x, axis=axis, keepdims=True)
    e = np.exp(x - m)
    return e / np.sum(e, axis=axis, keepdims=True)


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def log_beta(a, b):
    """ln B(a, b) of Eq. 3: B(a,b) = int_0^1 t^(a-1)(1-t)^(b-1) dt
    = Gamma(a)Gamma(b)/Gamma(a+b).  Pinned by closed forms lnB(1,1)=0, lnB(2,2)=-ln 6
     and by quadrature of Eq. 3's integral."""
    a = f64(a)
    b = f64(b)
    return gammaln(a) + gammaln(b) - gammaln(a + b)


def kl_beta(a1, b1, a2, b2):
    """KL( Beta(a1,b1) || Beta(a2,b2) ) per element, closed form (Eq. 3 densities).

    KL = lnB(a2,b2) - lnB(a1,b1) + (a1-a2) psi(a1) + (b1-b2) psi(b1)
         + (a2-a1+b2-b1) psi(a1+b1).
    Pinned by the closed forms KL(B(1,1)||B(2,2)) = 2 - ln 6, KL(B(2,2)||B(1,1))
    = ln 6 - 5/3 (fixes the direction), KL(p||p)=0, by adaptive quadrature of
    int p ln(p/q), and by torch.distributions.kl_divergence in float64."""
    a1, b1, a2, b2 = f64(a1), f64(b1), f64(a2), f64(b2)
    return (log_beta(a2, b2) - log_beta(a1, b1)
            + (a1 - a2) * digamma(a1) + (b1 - b2) * digamma(b1)
            + (a2 - a1 + b2 - b1) * digamma(a1 + b1))


def beta_regularizer(x):
    """Q2/Q12 [ext]: clamp(x + 1, 0.05, 1e9)."""
    return np.clip(f64(x) + REG_ADD, REG_MIN, REG_MAX)


# ----------------------------------------------------------------------------------------
# Model parameter views (fp32 tables from synth, promoted to float64 on use)
# ----------------------------------------------------------------------------------------
class Model:
    """Holds one model's tables. ``tables`` uses synth's names ('entity', 'relation',
    'offset', 'W:<layer>', 'b:<layer>')."""

    def __init__(self, kind, tables, dim, n_layers=2, terminal=TERMINAL_REGULARIZER):
        if kind not in ("gqe", "q2b", "betae"):
            raise ValueError(kind)
        self.kind = kind
        self.t = tables
        self.d = dim
        self.n_layers = n_layers
        self.terminal = terminal

    def W(self, name):
        return self.t["W:" + name], self.t["b:" + name]

    # ---- a2: anchor / relation gather ------------------------------------------------
    def anchor(self, ids):
        """Entity rows E[a].  GQE: q; Q2B: (center, offset=0); BetaE: regularised [alpha;beta]
        (Q12)."""
        e = f64(self.t["entity"][ids])
        if self.kind == "gqe":
            return e
        if self.kind == "q2b":
            return np.concatenate([e, np.zeros_like(e)], axis=-1)
        return beta_regularizer(e)

    # ---- a3: projection p ------------------------------------------------------------
    def project(self, x, rel_ids):
        """Relation projection ("S' = MLP_r(S)" for BetaE; [ext] for GQE/Q2B).
        GQE: q + R[r].  Q2B: (c + R_c[r], o + R_o[r]) (Q11: identity offset activation).
        BetaE: z = [alpha; beta; R[r]]; h = ReLU(W_l h + b_l) for l = 1..L;
        y = W_0 h + b_0; terminal (Q2): clamp(y+1, .05, 1e9) or Eq.-4 softmax."""
        r = f64(self.t["relation"][rel_ids])
        d = self.d
        if self.kind == "gqe":
            return x + r
        if self.kind == "q2b":
            ro = f64(self.t["offset"][rel_ids])
            return np.concatenate([x[..., :d] + r, x[..., d:] + ro], axis=-1)
        h = np.concatenate([x, r], axis=-1)                     # Eq. 4 var_S (with r) [Q3]
        for l in range(1, self.n_layers + 1):
            W, b = self.W(f"proj.layer{l}")
            h = relu(linear(h, W, b))                           # Eq. 4 matmul, add, relu
        W, b = self.W("proj.layer0")
        y = linear(h, W, b)                                     # Eq. 4 t7, t8
        if self.terminal == TERMINAL_SOFTMAX:
            return np.maximum(softmax(y, axis=-1), SOFTMAX_FLOOR)  # Eq. 4 var_S'
        return beta_regularizer(y)

    # ---- a4: negation n ---------------------------------------------------------------
    def negate(self, x):
        """Q5 [ext]: BetaE negation, alpha -> 1/alpha, beta -> 1/beta; no clamp after."""
        if self.kind != "betae":
            raise NotImplementedError("GQE/Q2B do not support the n operator (P:423)")
        return 1.0 / x

    # ---- a5: intersection i ----------------------------------------------------------
    def intersect(self, xs):
        """Q6 [ext]: attention over branches, softmax over the BRANCH axis per dimension.

        GQE / Q2B center:  s_i = W2 ReLU(W1 x_i + b1) + b2;  a = softmax_i(s);  sum_i a_i x_i.
        BetaE: input [alpha_i; beta_i] (2d) -> 2d -> d; the same a weights alpha and beta.
        Q2B offset: g = sigmoid(V2 mean_i ReLU(V1 o_i + c1) + c2);  o = min_i o_i * g.
        Pinned by: identical branches -> input; zero weights -> arithmetic mean; output in
        [min_i, max_i]; permutation invariance; Q2B zero weights -> min/2 (test_oracle_ops)."""
        X = np.stack(xs, axis=0)                                # [n, B, emb]
        d = self.d
        W1, b1 = self.W("inter.layer1")
        W2, b2 = self.W("inter.layer2")
        if self.kind == "gqe":
            att = softmax(linear(relu(linear(X, W1, b1)), W2, b2), axis=0)
            return np.sum(att * X, axis=0)
        if self.kind == "q2b":
            C = X[..., :d]
            O = X[..., d:]
            att = softmax(linear(relu(linear(C, W1, b1)), W2, b2), axis=0)
            c = np.sum(att * C, axis=0)
            V1, c1 = self.W("offset.layer1")
            V2, c2 = self.W("offset.layer2")
            g = sigmoid(linear(np.mean(relu(linear(O, V1, c1)), axis=0), V2, c2))
            o = np.min(O, axis=0) * g
            return np.concatenate([c, o], axis=-1)
        att = softmax(linear(relu(linear(X, W1, b1)), W2, b2), axis=0)   # [n, B, d]
        alpha = np.sum(att * X[..., :d], axis=0)
        beta = np.sum(att * X[..., d:], axis=0)
        return np.concatenate([alpha, beta], axis=-1)

    # ---- plan evaluation (Eq. 1 DNF; Eq. 2 mapping) -----------------------------------
    def embed(self, node, anchors, rels):
        k = node[0]
        if k == A:
            return self.anchor(anchors[:, node[1]])
        if k == P:
            return self.project(self.embed(node[1], anchors, rels), rels[:, node[2]])
        if k == N:
            return self.negate(self.embed(node[1], anchors, rels))
        if k == I:
            return self.intersect([self.embed(c, anchors, rels) for c in node[1]])
        raise ValueError("union is only allowed at the top level (DNF, Eq. 1)")

    def query_embedding(self, structure, anchors, rels):
        """[B, n_branches, emb] float64 with emb = d (GQE), 2d (Q2B: [center; offset]),
        2d (BetaE: [alpha; beta]).  2u/up: one embedding per DNF clause (Q7)."""
        if structure not in PLANS:
            raise ValueError(f"unknown structure {structure!r}; valid: {', '.join(STRUCTURES)}")
        if uses_negation(structure) and self.kind != "betae":
            raise NotImplementedError("GQE/Q2B do not support the n operator (P:423)")
        anchors = np.asarray(anchors)
        rels = np.asarray(rels)
        plan = PLANS[structure]
        if plan[0] == U:
            bs = [self.embed(c, anchors, rels) for c in plan[1]]
        else:
            bs = [self.embed(plan, anchors, rels)]
        return np.stack(bs, axis=1)

    # ---- a7: distances -----------------------------------------------------------------
    def entity_view(self, rows=None):
        e = self.t["entity"] if rows is None else self.t["entity"][rows]
        e = f64(e)
        return beta_regularizer(e) if self.kind == "betae" else e

    def distance(self, q, ent):
        """Distance between query embeddings q [B, emb] and entity rows ent [N, ...]
        (already in model view) -> [B, N].  Q8 [ext]:
        GQE  sum_d |e - q|;
        Q2B  sum_d ReLU(|e - c| - o) + cen * sum_d min(|e - c|, o);
        BetaE sum_d |KL(Beta(e) || Beta(q))| (entity first, torch norm p=1), literal
        per-(q, e, d) closed form (no entity/query decomposition)."""
        d = self.d
        if self.kind == "gqe":
            return np.sum(np.abs(ent[None, :, :] - q[:, None, :]), axis=-1)
        if self.kind == "q2b":
            c = q[:, None, :d]
            o = q[:, None, d:]
            delta = np.abs(ent[None, :, :] - c)
            out = np.maximum(delta - o, 0.0)
            inn = np.minimum(delta, o)
            return np.sum(out, axis=-1) + Q2B_CEN * np.sum(inn, axis=-1)
        kl = kl_beta(ent[None, :, :d], ent[None, :, d:], q[:, None, :d], q[:, None, d:])
        return np.sum(np.abs(kl), axis=-1)

    def scores(self, structure, anchors, rels, rows=None, chunk=None):
        """a6+a7: distance of every query to every entity (or entity ``rows``), min over DNF
        branches (Q7: max logit = min distance).  [B, N] float64."""
        qe = self.query_embedding(structure, anchors, rels)
        ent = self.entity_view(rows)
        B = qe.shape[0]
        out = np.empty((B, ent.shape[0]), np.float64)
        step = chunk or max(1, int(2e7 // max(1, ent.size)))
        for b0 in range(0, B, step):
            b1 = min(B, b0 + step)
            dist = None
            for br in range(qe.shape[1]):
                db = self.distance(qe[b0:b1, br, :], ent)
                dist = db if dist is None else np.minimum(dist, db)
            out[b0:b1] = dist
        return out


# ----------------------------------------------------------------------------------------
# a8: top-k with (distance ascending, entity id ascending) order (Q13; S:457 tie-break)
# ----------------------------------------------------------------------------------------
def topk(dist, k, ids=None):
    """Full sort of each row by (dist, id); returns (dist [B,k], id [B,k]) with global ids.
    Pinned by brute force on tiny inputs (test_oracle_ops)."""
    dist = np.asarray(dist)
    B, n = dist.shape
    ids = np.arange(n, dtype=np.int64) if ids is None else np.asarray(ids, np.int64)
    k = min(k, n)
    od = np.empty((B, k), np.float64)
    oi = np.empty((B, k), np.int64)
    for b in range(B):
        order = np.lexsort((ids, dist[b]))[:k]
        od[b] = dist[b, order]
        oi[b] = ids[order]
    return od, oi


def shard_range(n_entity, world, rank):
    """a9 / SURVEY §8(e): contiguous ranges, rank r owns [r*ceil(N/W), min(N,(r+1)*ceil(N/W)))."""
    per = -(-n_entity // world)
    return min(n_entity, rank * per), min(n_entity, (rank + 1) * per)


def merge_topk(parts_dist, parts_id, k):
    """a9: merge W per-shard top-k lists ([W,B,k] each) into the global top-k, (dist, id) order."""
    pd = np.concatenate(list(parts_dist), axis=1)
    pi = np.concatenate(list(parts_id), axis=1)
    B = pd.shape[0]
    od = np.empty((B, k), np.float64)
    oi = np.empty((B, k), np.int64)
    for b in range(B):
        order = np.lexsort((pi[b], pd[b]))[:k]
        od[b] = pd[b, order]
        oi[b] = pi[b, order]
    return od, oi


def answer(model, structure, anchors, rels, k):
    """Whole path a1..a8 on one batch: (topk_dist, topk_id, full dist)."""
    dist = model.scores(structure, anchors, rels)
    td, ti = topk(dist, k)
    return td, ti, dist


# ----------------------------------------------------------------------------------------
# N1: filtered ranking and MRR -- the accuracy check of RQ3,
# KGReasoning test protocol [ext]: entities ordered by distance (logit descending), each hard
# answer's rank counts only the NON-answer entities ranked before it ("filtered" setting);
# ties are broken by ascending entity id (Q13), as in top-k.
# ----------------------------------------------------------------------------------------
def filtered_ranks(dist_row, answers, ids=None):
    """dist_row: distances of one query to the entities `ids` (default 0..n-1); answers: all
    answers (easy and hard) of the query.  Returns {answer: 1 + #{e not in answers:
    (dist_e, e) < (dist_a, a)}} for every answer.  Pinned by an explicit full sort
    (test_oracle_ranking) and the SPEC S:465-473 MRR examples."""
    dist_row = np.asarray(dist_row, np.float64)
    ids = np.arange(len(dist_row), dtype=np.int64) if ids is None else np.asarray(ids, np.int64)
    pos = {int(e): i for i, e in enumerate(ids)}
    ans = set(int(a) for a in answers)
    keep = np.array([int(e) not in ans for e in ids])
    d_keep, id_keep = dist_row[keep], ids[keep]
    out = {}
    for a in ans:
        da = dist_row[pos[a]]
        better = (d_keep < da) | ((d_keep == da) & (id_keep < a))
        out[a] = 1 + int(np.count_nonzero(better))
    return out


def mrr_hits(ranks):
    """ranks: filtered ranks of the hard answers of one query -> (MRR, Hits@1, Hits@3, Hits@10),
    each a mean over those answers (KGReasoning averages per query)."""
    r = np.asarray(list(ranks), np.float64)
    return float(np.mean(1.0 / r)), float(np.mean(r <= 1)), float(np.mean(r <= 3)), float(np.mean(r <= 10))
