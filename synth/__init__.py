"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no projection, intersection,
negation, union, distance or ranking).  It only draws random numbers and builds
integer index arrays, so both sides of every parity check consume the exact
same fp32 tables and int32 queries (SURVEY.md §8(d) "Synthetic inputs").

Recipes (DESIGN.md §"Input recipe"):
  * ``kgr-init`` (default, "random-init weights" of BASELINE.json north_star):
      entity / relation rows  U(-(gamma+2)/d, +(gamma+2)/d)      [KGReasoning init, ext]
      Q2B relation offsets    U(0, (gamma+2)/d)
      nn.Linear weights       xavier_uniform U(+-sqrt(6/(fan_in+fan_out)))
      nn.Linear biases        U(+-1/sqrt(fan_in))                 [torch default]
  * ``spread`` (numeric stress): BetaE raw rows U(-0.95, 4.0) so that after the
      regulariser alpha,beta in [0.05, 5]; GQE/Q2B rows U(-1, 1); offsets U(0, 1).
Draws are float64 from ``numpy.random.default_rng(seed)`` rounded once to fp32.
Queries: anchors U{0..N-1}, relations U{0..R-1}, iid per slot (throughput).
(The planted integer KG used by brute-force tests lives in tests/planted.py.)
"""
from __future__ import annotations

import numpy as np

MODELS = ("gqe", "q2b", "betae")

# KGReasoning margins gamma; only used for the init range here.
INIT_GAMMA = {"gqe": 24.0, "q2b": 24.0, "betae": 60.0}
INIT_EPSILON = 2.0

# Slot counts per structure (SURVEY §8(b) slot table).  Pure bookkeeping.
STRUCTURES = ("1p", "2p", "3p", "2i", "3i", "pi", "ip", "2u", "up",
              "2in", "3in", "inp", "pin", "pni")
EPFO = STRUCTURES[:9]
NEGATION = STRUCTURES[9:]
#: De Morgan unions (BetaE only): not in the 14 benchmark types
DM = ("2u-DM", "up-DM")
ALL_STRUCTURES = STRUCTURES + DM
N_ANCHORS = {"1p": 1, "2p": 1, "3p": 1, "2i": 2, "3i": 3, "pi": 2, "ip": 2, "2u": 2,
             "up": 2, "2in": 2, "3in": 3, "inp": 2, "pin": 2, "pni": 2, "2u-DM": 2, "up-DM": 2}
N_RELS = {"1p": 1, "2p": 2, "3p": 3, "2i": 2, "3i": 3, "pi": 3, "ip": 3, "2u": 2,
          "up": 3, "2in": 2, "3in": 3, "inp": 3, "pin": 3, "pni": 3, "2u-DM": 2, "up-DM": 3}

# Canonical parameter names.  nn.Linear convention: W is [out_features, in_features].
#   betae: proj.layer1 [H,3d], proj.layer2..L [H,H], proj.layer0 [2d,H],
#          inter.layer1 [2d,2d], inter.layer2 [d,2d]
#   gqe:   inter.layer1 [d,d], inter.layer2 [d,d]
#   q2b:   inter.layer1/2 [d,d] (center net), offset.layer1/2 [d,d]


def _u(rng, lo, hi, shape):
    return rng.uniform(lo, hi, size=shape).astype(np.float32)


def _linear(rng, out_f, in_f):
    a = np.sqrt(6.0 / (in_f + out_f))
    w = _u(rng, -a, a, (out_f, in_f))
    bb = 1.0 / np.sqrt(in_f)
    b = _u(rng, -bb, bb, (out_f,))
    return w, b


def linear_shapes(model: str, d: int, hidden: int = 1600, n_layers: int = 2):
    """{name: (out_f, in_f)} for every nn.Linear the model owns."""
    if model == "betae":
        s = {"proj.layer1": (hidden, 3 * d)}
        for l in range(2, n_layers + 1):
            s[f"proj.layer{l}"] = (hidden, hidden)
        s["proj.layer0"] = (2 * d, hidden)
        s["inter.layer1"] = (2 * d, 2 * d)
        s["inter.layer2"] = (d, 2 * d)
        return s
    if model == "gqe":
        return {"inter.layer1": (d, d), "inter.layer2": (d, d)}
    if model == "q2b":
        return {"inter.layer1": (d, d), "inter.layer2": (d, d),
                "offset.layer1": (d, d), "offset.layer2": (d, d)}
    raise ValueError(model)


def make_tables(model: str, n_entity: int, n_relation: int, dim: int, *,
                hidden: int = 1600, n_layers: int = 2, seed: int = 2503_02172,
                dist: str = "kgr-init", entity_rows: tuple[int, int] | None = None):
    """Return a dict of fp32 arrays: entity, relation, [offset], and 'W:<name>', 'b:<name>'.

    ``entity_rows=(lo, hi)`` draws only that slice of the entity table, with the
    same values as the full draw (entity rows come from a per-row-block stream),
    so a 2M-entity shard can be generated without materialising the others.
    """
    if model not in MODELS:
        raise ValueError(f"model must be one of {MODELS}")
    rng = np.random.default_rng(seed)
    rng_w = np.random.default_rng(seed + 17)
    t: dict[str, np.ndarray] = {}
    ew = 2 * dim if model == "betae" else dim
    rnge = (INIT_GAMMA[model] + INIT_EPSILON) / dim
    if dist == "kgr-init":
        lo, hi = -rnge, rnge
    elif dist == "spread":
        lo, hi = (-0.95, 4.0) if model == "betae" else (-1.0, 1.0)
    else:
        raise ValueError(dist)
    t["entity"] = _entity_block_draw(seed, n_entity, ew, lo, hi, entity_rows)
    t["relation"] = _u(rng, -rnge if dist == "kgr-init" else -1.0,
                       rnge if dist == "kgr-init" else 1.0, (n_relation, dim))
    if model == "q2b":
        t["offset"] = _u(rng, 0.0, rnge if dist == "kgr-init" else 1.0, (n_relation, dim))
    for name, (o, i) in linear_shapes(model, dim, hidden, n_layers).items():
        w, b = _linear(rng_w, o, i)
        t["W:" + name] = w
        t["b:" + name] = b
    return t


_BLOCK = 65536


def _entity_block_draw(seed, n, width, lo, hi, rows):
    lo_r, hi_r = (0, n) if rows is None else rows
    out = np.empty((hi_r - lo_r, width), np.float32)
    b0 = lo_r // _BLOCK
    b1 = (hi_r + _BLOCK - 1) // _BLOCK
    for b in range(b0, b1):
        r0 = b * _BLOCK
        r1 = min(n, r0 + _BLOCK)
        blk = np.random.default_rng([seed, 1, b]).uniform(lo, hi, size=(r1 - r0, width))
        s0 = max(r0, lo_r)
        s1 = min(r1, hi_r)
        out[s0 - lo_r:s1 - lo_r] = blk[s0 - r0:s1 - r0].astype(np.float32)
    return out


def make_queries(structure: str, batch: int, n_entity: int, n_relation: int, seed: int):
    """Uniform throughput queries: anchors int32 [B, n_a], rels int32 [B, n_r]."""
    if structure not in ALL_STRUCTURES:
        raise ValueError(f"unknown structure {structure!r}; valid: {', '.join(ALL_STRUCTURES)}")
    rng = np.random.default_rng(seed)
    a = rng.integers(0, n_entity, size=(batch, N_ANCHORS[structure]), dtype=np.int64)
    r = rng.integers(0, n_relation, size=(batch, N_RELS[structure]), dtype=np.int64)
    return a.astype(np.int32), r.astype(np.int32)


def query_seed(table_seed: int, structure: str) -> int:
    return table_seed + 1000 + ALL_STRUCTURES.index(structure)
