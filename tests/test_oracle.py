"""Pins for the float64 oracle (-m "not gpu").

Each test fixes a piece of the oracle against something other than the oracle itself:
closed forms, quadrature of Eq. 3, mpmath, torch library routines, invariants of the
operators, and brute force.  Chosen so that a plausible slip (dropped term, wrong sign or
KL direction, transposed weight, softmax over the wrong axis, mean vs sum, wrong plan
slot) fails at least one of them.
"""
import json
import os

import mpmath
import numpy as np
import pytest
import torch
from scipy import integrate

import oracle as O
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


# ------------------------------------------------------------------ special functions
@pytest.mark.parametrize("case", GOLD["log_beta"])
def test_log_beta_closed_forms(case):
    assert O.log_beta(case["a"], case["b"]) == pytest.approx(case["value"], abs=1e-14)


def test_log_beta_quadrature_and_symmetry():
    rng = np.random.default_rng(0)
    for _ in range(40):
        a, b = rng.uniform(1.0, 10.0, size=2)
        q, _ = integrate.quad(lambda t: t ** (a - 1) * (1 - t) ** (b - 1), 0, 1, limit=400,
                              epsabs=1e-14, epsrel=1e-12)
        assert O.log_beta(a, b) == pytest.approx(np.log(q), abs=1e-9)
        assert O.log_beta(a, b) == pytest.approx(O.log_beta(b, a), abs=1e-14)


def test_digamma_against_closed_forms_and_mpmath():
    from scipy.special import digamma
    for c in GOLD["digamma"]:
        assert digamma(c["x"]) == pytest.approx(c["value"], abs=1e-14)
    for x in np.geomspace(0.05, 50, 37):
        assert digamma(x) == pytest.approx(float(mpmath.digamma(x)), rel=1e-12, abs=1e-13)


@pytest.mark.parametrize("case", GOLD["kl_beta"])
def test_kl_beta_closed_forms(case):
    (a1, b1), (a2, b2) = case["entity"], case["query"]
    assert O.kl_beta(a1, b1, a2, b2) == pytest.approx(case["value"], abs=1e-12)


def test_kl_beta_quadrature_and_torch():
    rng = np.random.default_rng(1)
    for _ in range(30):
        a1, b1, a2, b2 = rng.uniform(0.3, 8.0, size=4)
        lp = lambda x, a, b: (a - 1) * np.log(x) + (b - 1) * np.log1p(-x) - O.log_beta(a, b)
        f = lambda x: np.exp(lp(x, a1, b1)) * (lp(x, a1, b1) - lp(x, a2, b2))
        q, _ = integrate.quad(f, 0, 1, limit=400, epsabs=1e-13, epsrel=1e-11)
        v = O.kl_beta(a1, b1, a2, b2)
        assert v == pytest.approx(q, rel=1e-7, abs=1e-9)
        t = torch.distributions.kl_divergence(
            torch.distributions.Beta(torch.tensor(a1, dtype=torch.float64), torch.tensor(b1, dtype=torch.float64)),
            torch.distributions.Beta(torch.tensor(a2, dtype=torch.float64), torch.tensor(b2, dtype=torch.float64)))
        assert v == pytest.approx(float(t), rel=1e-12, abs=1e-13)
        assert v >= 0


# ------------------------------------------------------------------ small model helpers
def tiny_tables(model, n=40, r=6, d=8, hidden=16, layers=2, seed=3, dist="kgr-init"):
    return synth.make_tables(model, n, r, d, hidden=hidden, n_layers=layers, seed=seed, dist=dist)


def test_linear_matches_torch():
    rng = np.random.default_rng(2)
    W = rng.standard_normal((5, 3)).astype(np.float32)
    b = rng.standard_normal(5).astype(np.float32)
    x = rng.standard_normal((4, 3)).astype(np.float32)
    ref = torch.nn.functional.linear(torch.tensor(x, dtype=torch.float64),
                                     torch.tensor(W, dtype=torch.float64),
                                     torch.tensor(b, dtype=torch.float64)).numpy()
    np.testing.assert_allclose(O.linear(x, W, b), ref, rtol=0, atol=1e-14)


def test_gqe_1p_worked_example():
    g = GOLD["gqe_1p"]
    t = {"entity": np.array([g["entity_anchor"]] + g["targets"], np.float32),
         "relation": np.array([g["relation"]], np.float32)}
    m = O.Model("gqe", t, dim=2)
    q = m.query_embedding("1p", np.array([[0]]), np.array([[0]]))
    np.testing.assert_array_equal(q[0, 0], g["query"])
    d = m.scores("1p", np.array([[0]]), np.array([[0]]))[0]
    np.testing.assert_allclose(d[1:], g["dist"], atol=0)


def test_q2b_box_distance_worked_example():
    g = GOLD["q2b_box"]
    m = O.Model("q2b", {"entity": np.zeros((1, 1), np.float32)}, dim=1)
    q = np.array([g["center"] + g["offset"]], np.float64)
    d = m.distance(q, np.array(g["entities"], np.float64))[0]
    np.testing.assert_allclose(d, g["dist"], rtol=1e-14)


def betae_identity_mlp_tables():
    """GOLD betae_anchor_identity_mlp: d = 1, one hidden layer of width 2 that copies
    [alpha; beta] (W1 = [[1,0,0],[0,1,0]]), W0 = I2, zero biases, zero attention weights."""
    g = GOLD["betae_anchor_identity_mlp"]
    t = synth.make_tables("betae", 3, 1, 1, hidden=2, n_layers=1, seed=1)
    t["entity"] = np.array(g["entity_raw"], np.float32)
    t["relation"][:] = 0.7            # must not leak into the output: W1's relation column is 0
    t["W:proj.layer1"] = np.array([[1, 0, 0], [0, 1, 0]], np.float32)
    t["W:proj.layer0"] = np.eye(2, dtype=np.float32)
    for k in list(t):
        if k.startswith("b:") or k.startswith("W:inter"):
            t[k] = np.zeros_like(t[k])
    return g, O.Model("betae", t, dim=1, n_layers=1)


def test_betae_anchor_regulariser_worked_example():
    """Q12 pin (Eq. 3: Beta parameters > 0): anchors are the regularised entity rows
    clamp(x + 1, 0.05, 1e9) -- raw 1.0 -> 2.0, raw -3.0 -> 0.05 (floor), raw 0.5 -> 1.5 -- and
    an identity-copy MLP shows them through the projection terminal (clamp(y + 1)): a missing
    or doubled anchor regulariser changes every value below."""
    g, m = betae_identity_mlp_tables()
    np.testing.assert_array_equal(m.anchor(np.arange(3)), np.array(g["anchor_view"]))
    assert m.anchor(np.array([1]))[0, 0] == 0.05 and m.anchor(np.array([0]))[0, 0] == 2.0
    q = m.query_embedding("1p", np.arange(3)[:, None], np.zeros((3, 1), np.int64))[:, 0]
    np.testing.assert_allclose(q, np.array(g["query_1p"]), rtol=1e-15)
    d = m.scores("1p", np.array([[0]]), np.array([[0]]))[0, 0]   # KL(Beta(2,2) || Beta(3,3))
    assert d == pytest.approx(g["dist_1p_anchor0_to_entity0"], rel=1e-13)
    two = g["query_2i_zero_attention"]
    q2 = m.query_embedding("2i", np.array([two["anchors"]]), np.zeros((1, 2), np.int64))[0, 0]
    np.testing.assert_allclose(q2, two["value"], rtol=1e-15)
    # identical Beta(2,2) anchors through 2i -> the 1p embedding Beta(3,3)
    q3 = m.query_embedding("2i", np.array([[0, 0]]), np.zeros((1, 2), np.int64))[0, 0]
    np.testing.assert_allclose(q3, [3.0, 3.0], rtol=1e-15)


def test_q2b_offset_projection_worked_example():
    """Q11 pin: the Q2B projection translates the box, (c, o) -> (c + R_c[r], o + R_o[r]) with
    the identity offset activation and a zero anchor offset (Q10); hand-worked 1p / 2p boxes
    and box distances (GOLD q2b_offset_projection)."""
    g = GOLD["q2b_offset_projection"]
    t = synth.make_tables("q2b", 5, 2, 2, seed=1)
    t["entity"] = np.array(g["entity"], np.float32)
    t["relation"] = np.array(g["relation"], np.float32)
    t["offset"] = np.array(g["offset"], np.float32)
    m = O.Model("q2b", t, dim=2)
    q1 = m.query_embedding("1p", np.array([[0]]), np.array([[0]]))[0, 0]
    np.testing.assert_allclose(q1, g["box_1p"], rtol=1e-7)
    np.testing.assert_allclose(m.scores("1p", np.array([[0]]), np.array([[0]]))[0], g["dist_1p"], rtol=1e-6)
    q2 = m.query_embedding("2p", np.array([[0]]), np.array([[0, 1]]))[0, 0]
    np.testing.assert_allclose(q2, g["box_2p"], rtol=1e-7)
    d2 = m.scores("2p", np.array([[0]]), np.array([[0, 1]]))[0]
    np.testing.assert_allclose(d2[g["dist_2p_entities"]], g["dist_2p"], rtol=1e-6, atol=1e-7)


def test_q2b_zero_offsets_equals_gqe_l1():
    t = tiny_tables("q2b")
    t["offset"][:] = 0
    m = O.Model("q2b", t, dim=8)
    g = O.Model("gqe", {"entity": t["entity"], "relation": t["relation"]}, dim=8)
    a, r = synth.make_queries("2p", 5, 40, 6, 1)
    np.testing.assert_allclose(m.scores("2p", a, r), g.scores("2p", a, r), rtol=1e-14)


def test_q2b_identity_out_plus_in():
    # sum ReLU(delta-o) + sum min(delta,o) == sum delta for any reals
    rng = np.random.default_rng(4)
    m = O.Model("q2b", {"entity": np.zeros((1, 6), np.float32)}, dim=6)
    q = rng.standard_normal((3, 12))
    e = rng.standard_normal((7, 6))
    old = O.kgq_oracle.Q2B_CEN
    try:
        O.kgq_oracle.Q2B_CEN = 1.0
        d = m.distance(q, e)
    finally:
        O.kgq_oracle.Q2B_CEN = old
    ref = np.abs(e[None] - q[:, None, :6]).sum(-1)
    np.testing.assert_allclose(d, ref, rtol=1e-13)


@pytest.mark.parametrize("model", ["gqe", "q2b", "betae"])
@pytest.mark.parametrize("n", [2, 3])
def test_intersection_of_identical_inputs_returns_input(model, n):
    t = tiny_tables(model)
    m = O.Model(model, t, dim=8)
    x = m.anchor(np.array([3, 5, 7]))
    out = m.intersect([x] * n)
    d = 8
    if model == "q2b":
        np.testing.assert_allclose(out[:, :d], x[:, :d], rtol=1e-13)   # centers only (finding 7)
    else:
        np.testing.assert_allclose(out, x, rtol=1e-13)


@pytest.mark.parametrize("model", ["gqe", "betae", "q2b"])
def test_intersection_zero_weights_is_mean_and_bounded(model):
    t = tiny_tables(model)
    for k in list(t):
        if k.startswith(("W:inter", "b:inter", "W:offset", "b:offset")):
            t[k][:] = 0
    m = O.Model(model, t, dim=8)
    xs = [m.project(m.anchor(np.array([i, i + 1])), np.array([i % 6, (i + 2) % 6])) for i in range(3)]
    out = m.intersect(xs)
    X = np.stack(xs)
    d = 8
    if model == "q2b":
        np.testing.assert_allclose(out[:, :d], X[..., :d].mean(0), rtol=1e-13)
        np.testing.assert_allclose(out[:, d:], 0.5 * X[..., d:].min(0), rtol=1e-13)
    else:
        np.testing.assert_allclose(out, X.mean(0), rtol=1e-13)


@pytest.mark.parametrize("model", ["gqe", "betae", "q2b"])
def test_intersection_convex_hull_and_permutation(model):
    t = tiny_tables(model, dist="spread")
    m = O.Model(model, t, dim=8)
    xs = [m.project(m.anchor(np.arange(4) + 4 * i), np.arange(4) % 6) for i in range(3)]
    out = m.intersect(xs)
    X = np.stack(xs)
    cen = slice(0, 8) if model == "q2b" else slice(None)
    assert np.all(out[:, cen] >= X[..., cen].min(0) - 1e-12)
    assert np.all(out[:, cen] <= X[..., cen].max(0) + 1e-12)
    np.testing.assert_allclose(m.intersect(xs[::-1]), out, rtol=1e-12)
    np.testing.assert_allclose(m.intersect([xs[1], xs[2], xs[0]]), out, rtol=1e-12)
    if model == "q2b":  # 0 <= o_out <= min o_i for o_i >= 0
        assert np.all(out[:, 8:] >= 0) and np.all(out[:, 8:] <= X[..., 8:].min(0) + 1e-15)


def test_q2b_offset_gate_uses_mean_over_branches():
    # n identical offset branches: mean_i ReLU(V1 o + c1) is n-independent (sum would not be)
    t = tiny_tables("q2b")
    m = O.Model("q2b", t, dim=8)
    x = m.project(m.anchor(np.array([1, 2])), np.array([3, 4]))
    np.testing.assert_allclose(m.intersect([x, x])[:, 8:], m.intersect([x, x, x])[:, 8:], rtol=1e-13)


def test_betae_projection_zero_weights_gives_uniform_beta():
    t = tiny_tables("betae")
    for k in list(t):
        if k.startswith(("W:proj", "b:proj")):
            t[k][:] = 0
    m = O.Model("betae", t, dim=8)
    q = m.query_embedding("1p", np.array([[1]]), np.array([[2]]))
    np.testing.assert_array_equal(q, np.ones((1, 1, 16)))
    # entity raw row = 1 -> regularised Beta(2,2) in every dim: distance d * (ln 6 - 5/3)
    t["entity"][5] = 1.0
    d = m.scores("1p", np.array([[1]]), np.array([[2]]))[0, 5]
    assert d == pytest.approx(8 * (np.log(6) - 5 / 3), rel=1e-13)
    # bias-only output layer b0 = c -> constant Beta(clamp(c+1))
    t["b:proj.layer0"][:] = np.float32(0.5)
    q = m.query_embedding("1p", np.array([[1]]), np.array([[2]]))
    np.testing.assert_allclose(q, 1.5, rtol=0)
    t["b:proj.layer0"][:] = np.float32(-3.0)
    q = m.query_embedding("1p", np.array([[1]]), np.array([[2]]))
    np.testing.assert_allclose(q, 0.05, rtol=0)


def test_betae_projection_matches_torch_mlp():
    t = tiny_tables("betae", layers=3)
    m = O.Model("betae", t, dim=8, n_layers=3)
    x = m.anchor(np.array([0, 1, 2]))
    rid = np.array([1, 2, 3])
    tt = lambda a: torch.tensor(np.asarray(a), dtype=torch.float64)
    h = torch.cat([tt(x), tt(t["relation"][rid])], dim=-1)
    F = torch.nn.functional
    for l in (1, 2, 3):
        h = F.relu(F.linear(h, tt(t[f"W:proj.layer{l}"]), tt(t[f"b:proj.layer{l}"])))
    y = F.linear(h, tt(t["W:proj.layer0"]), tt(t["b:proj.layer0"]))
    ref = torch.clamp(y + 1, 0.05, 1e9).numpy()
    np.testing.assert_allclose(m.project(x, rid), ref, rtol=1e-13)
    ms = O.Model("betae", t, dim=8, n_layers=3, terminal=O.TERMINAL_SOFTMAX)
    sm = ms.project(x, rid)
    np.testing.assert_allclose(sm, np.maximum(torch.softmax(y, -1).numpy(), 1e-6), rtol=1e-13)
    np.testing.assert_allclose(sm.sum(-1), 1.0, rtol=1e-6)


def test_betae_intersection_matches_torch_module_semantics():
    # torch.distributions-free check of the shared-attention form: softmax over dim 0
    t = tiny_tables("betae", dist="spread")
    m = O.Model("betae", t, dim=8)
    xs = [m.anchor(np.array([i, i + 3])) for i in range(3)]
    X = torch.tensor(np.stack(xs))
    F = torch.nn.functional
    tt = lambda a: torch.tensor(a, dtype=torch.float64)
    s = F.linear(F.relu(F.linear(X, tt(t["W:inter.layer1"]), tt(t["b:inter.layer1"]))),
                 tt(t["W:inter.layer2"]), tt(t["b:inter.layer2"]))
    att = torch.softmax(s, dim=0)
    ref = torch.cat([(att * X[..., :8]).sum(0), (att * X[..., 8:]).sum(0)], -1).numpy()
    np.testing.assert_allclose(m.intersect(xs), ref, rtol=1e-13)


def test_negation_involution_and_example():
    m = O.Model("betae", tiny_tables("betae"), dim=8)
    x = m.anchor(np.arange(6))
    np.testing.assert_allclose(m.negate(m.negate(x)), x, rtol=2.3e-16)
    np.testing.assert_array_equal(m.negate(np.array([2.0, 0.5])), [0.5, 2.0])
    with pytest.raises(NotImplementedError):
        O.Model("gqe", tiny_tables("gqe"), dim=8).query_embedding("2in", np.zeros((1, 2), int), np.zeros((1, 2), int))


@pytest.mark.parametrize("model", ["gqe", "q2b", "betae"])
def test_union_is_min_over_dnf_branches(model):
    t = tiny_tables(model)
    m = O.Model(model, t, dim=8)
    a, r = synth.make_queries("up", 6, 40, 6, 9)
    d_up = m.scores("up", a, r)
    d1 = m.scores("2p", a[:, [0]], r[:, [0, 2]])
    d2 = m.scores("2p", a[:, [1]], r[:, [1, 2]])
    np.testing.assert_allclose(d_up, np.minimum(d1, d2), rtol=1e-15)
    a2, r2 = synth.make_queries("2u", 6, 40, 6, 10)
    np.testing.assert_allclose(m.scores("2u", a2, r2),
                               np.minimum(m.scores("1p", a2[:, [0]], r2[:, [0]]),
                                          m.scores("1p", a2[:, [1]], r2[:, [1]])), rtol=1e-15)
    same = np.concatenate([a2[:, [0]], a2[:, [0]]], 1), np.concatenate([r2[:, [0]], r2[:, [0]]], 1)
    np.testing.assert_allclose(m.scores("2u", *same), m.scores("1p", a2[:, [0]], r2[:, [0]]), rtol=1e-15)


@pytest.mark.parametrize("model", ["gqe", "betae"])
def test_structure_reductions(model):
    t = tiny_tables(model)
    m = O.Model(model, t, dim=8)
    a, r = synth.make_queries("1p", 5, 40, 6, 11)
    aa, rr = np.repeat(a, 2, 1), np.repeat(r, 2, 1)
    np.testing.assert_allclose(m.query_embedding("2i", aa, rr), m.query_embedding("1p", a, r), rtol=1e-13)
    # ip = projection of the 2i embedding by slot 2
    a3, r3 = synth.make_queries("ip", 5, 40, 6, 12)
    e2i = m.query_embedding("2i", a3, r3[:, :2])[:, 0]
    np.testing.assert_allclose(m.query_embedding("ip", a3, r3)[:, 0], m.project(e2i, r3[:, 2]), rtol=1e-13)
    # pi = I(2p(a0; r0 r1), 1p(a1; r2))
    e_a = m.query_embedding("2p", a3[:, [0]], r3[:, [0, 1]])[:, 0]
    e_b = m.query_embedding("1p", a3[:, [1]], r3[:, [2]])[:, 0]
    np.testing.assert_allclose(m.query_embedding("pi", a3, r3)[:, 0], m.intersect([e_a, e_b]), rtol=1e-13)


def test_negation_structure_layouts():
    t = tiny_tables("betae")
    m = O.Model("betae", t, dim=8)
    a, r = synth.make_queries("pni", 4, 40, 6, 13)
    p1 = lambda ai, ri: m.query_embedding("1p", a[:, [ai]], r[:, [ri]])[:, 0]
    p2 = lambda ai, r0, r1: m.query_embedding("2p", a[:, [ai]], r[:, [r0, r1]])[:, 0]
    np.testing.assert_allclose(m.query_embedding("pni", a, r)[:, 0],
                               m.intersect([m.negate(p2(0, 0, 1)), p1(1, 2)]), rtol=1e-13)
    np.testing.assert_allclose(m.query_embedding("pin", a, r)[:, 0],
                               m.intersect([p2(0, 0, 1), m.negate(p1(1, 2))]), rtol=1e-13)
    e2in = m.query_embedding("2in", a, r[:, :2])[:, 0]
    np.testing.assert_allclose(m.query_embedding("2in", a, r[:, :2])[:, 0],
                               m.intersect([p1(0, 0), m.negate(p1(1, 1))]), rtol=1e-13)
    np.testing.assert_allclose(m.query_embedding("inp", a, r)[:, 0], m.project(e2in, r[:, 2]), rtol=1e-13)
    a3, r3 = synth.make_queries("3in", 4, 40, 6, 14)
    q = lambda i: m.query_embedding("1p", a3[:, [i]], r3[:, [i]])[:, 0]
    np.testing.assert_allclose(m.query_embedding("3in", a3, r3)[:, 0],
                               m.intersect([q(0), q(1), m.negate(q(2))]), rtol=1e-13)


def test_de_morgan_union_pins():
    """N4 (2u-DM / up-DM, N(I(N x, N y))): identical branches reduce to 1p / 2p (intersection
    of identical inputs returns it, negation is an involution); with zero intersection weights
    the attention is uniform, so 2u-DM is the element-wise HARMONIC mean of the two branch
    embeddings (1 / mean(1/x_i)) -- a closed form that a missing outer or inner negation, or an
    arithmetic mean, fails; branch order does not matter; GQE/Q2B reject it."""
    t = tiny_tables("betae", dist="spread")
    m = O.Model("betae", t, dim=8)
    a, r = synth.make_queries("up-DM", 5, 40, 6, 21)
    p1 = lambda ai, ri: m.query_embedding("1p", a[:, [ai]], r[:, [ri]])[:, 0]
    same_a, same_r = np.repeat(a[:, [0]], 2, 1), np.repeat(r[:, [0]], 2, 1)
    np.testing.assert_allclose(m.query_embedding("2u-DM", same_a, same_r)[:, 0], p1(0, 0), rtol=1e-12)
    same_r3 = np.concatenate([r[:, [0, 0]], r[:, [2]]], 1)
    np.testing.assert_allclose(m.query_embedding("up-DM", same_a, same_r3)[:, 0],
                               m.query_embedding("2p", a[:, [0]], r[:, [0, 2]])[:, 0], rtol=1e-12)
    swap = m.query_embedding("2u-DM", a[:, ::-1], r[:, [1, 0]])[:, 0]
    np.testing.assert_allclose(swap, m.query_embedding("2u-DM", a, r[:, :2])[:, 0], rtol=1e-12)
    # up-DM = P(2u-DM, r2)
    np.testing.assert_allclose(m.query_embedding("up-DM", a, r)[:, 0],
                               m.project(m.query_embedding("2u-DM", a, r[:, :2])[:, 0], r[:, 2]), rtol=1e-13)
    t0 = tiny_tables("betae", dist="spread")
    for k in list(t0):
        if k.startswith(("W:inter", "b:inter")):
            t0[k][:] = 0
    m0 = O.Model("betae", t0, dim=8)
    x = m0.query_embedding("1p", a[:, [0]], r[:, [0]])[:, 0]
    y = m0.query_embedding("1p", a[:, [1]], r[:, [1]])[:, 0]
    np.testing.assert_allclose(m0.query_embedding("2u-DM", a, r[:, :2])[:, 0], 2.0 / (1.0 / x + 1.0 / y),
                               rtol=1e-13)
    assert O.kgq_oracle.uses_negation("2u-DM") and O.kgq_oracle.n_branches("up-DM") == 1
    with pytest.raises(NotImplementedError):
        O.Model("q2b", tiny_tables("q2b"), dim=8).query_embedding("2u-DM", a, r[:, :2])


def test_slot_counts_match_synth():
    for s in O.STRUCTURES:
        assert O.kgq_oracle.n_anchors(s) == synth.N_ANCHORS[s]
        assert O.kgq_oracle.n_relations(s) == synth.N_RELS[s]
        assert O.kgq_oracle.n_branches(s) == (2 if s in ("2u", "up") else 1)


def test_betae_self_query_ranks_first():
    # query equal to entity 7's embedding -> entity 7 first with KL 0
    t = tiny_tables("betae", dist="spread")
    m = O.Model("betae", t, dim=8)
    q = m.entity_view(np.array([7]))
    d = m.distance(q, m.entity_view())
    assert np.argmin(d[0]) == 7 and abs(d[0, 7]) < 1e-13


def test_topk_brute_force_and_ties():
    rng = np.random.default_rng(5)
    dist = rng.integers(0, 6, size=(7, 30)).astype(np.float64)   # many exact ties
    td, ti = O.topk(dist, 9)
    for b in range(7):
        pairs = sorted((dist[b, i], i) for i in range(30))[:9]
        assert [p[1] for p in pairs] == list(ti[b])
        assert [p[0] for p in pairs] == list(td[b])
    # k > n clamps; sharded merge equals global top-k
    W = 3
    parts = [O.topk(dist[:, slice(*O.shard_range(30, W, w))], 9,
                    ids=np.arange(*O.shard_range(30, W, w))) for w in range(W)]
    md, mi = O.merge_topk([p[0] for p in parts], [p[1] for p in parts], 9)
    np.testing.assert_array_equal(mi, ti)
    np.testing.assert_array_equal(md, td)


def test_shard_range_partitions():
    for n in (1, 7, 30, 14505, 2_000_000):
        for w in (1, 2, 3, 8):
            rs = [O.shard_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
