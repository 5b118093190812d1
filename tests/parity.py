"""Tolerance-aware comparators for GPU-vs-oracle parity.

Q14 per distance: |d_gpu - d_ref| <= rel * max(|d_ref|, s_q), s_q = 1e-3 * median_e d_ref(q)
    (near-zero distances -- planted exact matches, KL(p||p) -- are judged against the
    query's distance scale, because fp32 cancellation there is absolute).
Q15 top-k: tau = oracle k-th distance, tol = rel * max(tau, s_q).  Pass iff
    (i) every GPU id has oracle distance <= tau + tol;
    (ii) every id with oracle distance < tau - tol is present;
    (iii) GPU distances are non-decreasing, ids unique, each within Q14 of its oracle value;
    (iv) among GPU entries with equal GPU distance, ids ascend (the (dist, id) order).
"""
import numpy as np

REL = 1e-4  # BASELINE.json north_star: "within 1e-4 relative in fp32"


def row_scale(ref):
    return 1e-3 * np.median(ref, axis=-1, keepdims=True)


def assert_dist_close(got, ref, rel=REL, what=""):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    assert np.all(np.isfinite(got)), f"{what}: non-finite GPU distances"
    err = np.abs(got - ref) / np.maximum(np.abs(ref), row_scale(ref))
    worst = np.unravel_index(np.argmax(err), err.shape)
    assert err.max() <= rel, (f"{what}: max rel err {err.max():.3g} at {worst}: "
                              f"gpu {got[worst]!r} ref {ref[worst]!r}")
    return float(err.max())


def assert_embedding_close(got, ref, rel=REL, what="", floor=1e-3):
    """Element-wise |got - ref| <= rel * max(|ref|, floor * max_row |ref|)."""
    if isinstance(rel, tuple):  # (rel, floor) from chain_tolerance
        rel, floor = rel
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    floor = floor * np.max(np.abs(ref), axis=-1, keepdims=True)
    err = np.abs(got - ref) / np.maximum(np.abs(ref), floor)
    assert err.max() <= rel, f"{what}: max rel err {err.max():.3g}"
    return float(err.max())


def assert_topk_ok(gd, gi, ref_row, k, id_base=0, rel=REL, what="", sample_ids=None):
    """gd/gi: GPU top-k of one query; ref_row: oracle distances of this query over the ids
    [id_base, id_base + len(ref_row)) (the full row)."""
    gd = np.asarray(gd, np.float64)
    gi = np.asarray(gi, np.int64)
    loc = gi - id_base
    assert np.all((loc >= 0) & (loc < len(ref_row))), f"{what}: ids out of range {gi}"
    assert len(set(gi.tolist())) == k, f"{what}: duplicate ids {gi}"
    s_q = 1e-3 * np.median(ref_row)
    part = np.partition(ref_row, k - 1)[k - 1]
    tau = part
    tol = rel * max(tau, s_q)
    assert np.all(ref_row[loc] <= tau + tol), f"{what}: id with oracle dist > tau + tol"
    must = np.nonzero(ref_row < tau - tol)[0]
    assert set(must.tolist()) <= set(loc.tolist()), f"{what}: missing ids {set(must.tolist()) - set(loc.tolist())}"
    assert np.all(np.diff(gd) >= 0), f"{what}: distances not sorted"
    err = np.abs(gd - ref_row[loc]) / np.maximum(ref_row[loc], s_q)
    assert err.max() <= rel, f"{what}: top-k distance err {err.max():.3g}"
    eq = np.nonzero(np.diff(gd) == 0)[0]
    assert np.all(gi[eq] < gi[eq + 1]), f"{what}: ties not ordered by id"


def assert_topk_ok_sampled(gd, gi, ref_of_ids, sample_ids, ref_sample, k, rel=REL, what=""):
    """Size-independent top-k property for tables too large for a full oracle row:
    ref_of_ids = oracle distances of the returned ids; sample_ids / ref_sample = a random
    entity sample and its oracle distances.  Checks Q15 (iii) and that no sampled entity
    outside the returned set beats the returned k-th oracle distance by more than tol."""
    gd = np.asarray(gd, np.float64)
    gi = np.asarray(gi, np.int64)
    s_q = 1e-3 * np.median(ref_sample)
    assert len(set(gi.tolist())) == k, f"{what}: duplicate ids"
    assert np.all(np.diff(gd) >= 0), f"{what}: distances not sorted"
    err = np.abs(gd - ref_of_ids) / np.maximum(ref_of_ids, s_q)
    assert err.max() <= rel, f"{what}: top-k distance err {err.max():.3g}"
    tau = ref_of_ids.max()
    tol = rel * max(tau, s_q)
    outside = ~np.isin(np.asarray(sample_ids, np.int64), gi)
    assert np.all(ref_sample[outside] >= tau - tol), f"{what}: a sampled entity beats the k-th"


def chain_tolerance(structure, dist="kgr-init", model="betae", terminal="regularizer"):
    """(rel, floor) for intermediate query embeddings: element-wise
    |x_gpu - x_ref| <= rel * max(|x_ref|, floor * max_row |x_ref|).

    rel = 1e-4 -- the north-star bound -- for every structure without negation, both recipes.
    BetaE negation structures: an MLP output near the regulariser floor (y + 1 ~ 0.05) carries
    the GEMM's absolute error ~1.4e-7 sum|w h|; 1/x maps it to a Beta parameter ~20 with the same
    RELATIVE error (~1e-4 at K = 1600), which the attention softmax and the next projection
    propagate: rel = 2e-4; inp, whose post-intersection projection takes the negated (up to
    20) parameters as MLP input: 1e-3 at kgr-init, 2e-3 under 'spread' (alpha, beta in [0.05,
    5]).  Measured maxima (DRAIN 4): 2in/3in/pin/pni <= 1.0e-4, inp <= 7.3e-4 (kgr-init) /
    8.9e-4 (spread); profiles/r02/chain_err_drain.txt.  The literal Eq.-4 softmax terminal
    (KGQ_TERM_SOFTMAX) produces parameters down to its 1e-6 floor, so negation maps them to up
    to 1e6 and the same absolute GEMM error is amplified far more: 1e-3 for every negation
    structure there (measured 3.3e-4 for 2in).
    floor: BetaE parameters are >= 0.05, so the floor never binds there (1e-3).  GQE / Q2B
    coordinates change sign; an n-term fp32 sum errs by up to n u max|term| in ABSOLUTE terms
    (u = 2^-24), so next to a zero crossing the relative error is unbounded -- floor 1e-2 of the
    row max bounds it by 4 u / 1e-2 = 2.4e-5 for a 3-hop chain (measured <= 2.2e-5; with floor
    1e-3 the same cancellation measured up to 1.04e-4).  Distances are held to 1e-4 regardless."""
    floor = 1e-3 if model == "betae" else 1e-2
    negation = structure in ("2in", "3in", "inp", "pin", "pni", "2u-DM", "up-DM")
    if not negation:
        return 1e-4, floor
    if terminal == "softmax":
        return 1e-3, floor
    if structure == "inp":
        return (1e-3 if dist == "kgr-init" else 2e-3), floor
    return 2e-4, floor
