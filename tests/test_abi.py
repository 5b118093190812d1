"""CPU checks of the C ABI library: it loads, exports every symbol include/kgq.h declares,
and its pure-host entry points (structure metadata, shard ranges, argument validation) work
without a GPU.  No compute calls here."""
import ctypes
import os
import re

import pytest

import oracle as O
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
kgq = pytest.importorskip("paper_2503_02172_b200.kgq",
                          reason="libkgq.so not built (run __graft_entry__.build())")


def header_functions():
    src = open(os.path.join(ROOT, "include", "kgq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kgq_[a-z_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    names = header_functions()
    assert len(names) >= 25
    lib = ctypes.CDLL(kgq.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), f"{n} declared in kgq.h but not exported"
    assert set(names) == set(kgq.EXPORTS)


def test_both_operand_builds_export_every_symbol():
    """libkgq.so (fp16x2 GEMM operands) and libkgq_bf16x3.so (exact three-plane bf16 split) are
    the same ABI; kgq_tensor_mmas_per_fma tells them apart (3 vs 6 MMAs per fp32 multiply-add)."""
    here = os.path.dirname(kgq.LIB_PATH)
    mmas = {}
    for name in ("libkgq.so", "libkgq_bf16x3.so"):
        lib = ctypes.CDLL(os.path.join(here, name))
        for n in header_functions():
            assert hasattr(lib, n), f"{name}: {n} not exported"
        lib.kgq_tensor_mmas_per_fma.restype = ctypes.c_int32
        mmas[name] = lib.kgq_tensor_mmas_per_fma()
    assert mmas == {"libkgq.so": 3, "libkgq_bf16x3.so": 6}


def test_structure_metadata_matches_oracle_plans():
    for i, s in enumerate(O.STRUCTURES):
        assert kgq.structure_id(s) == i
        assert kgq.num_anchors(s) == synth.N_ANCHORS[s] == O.kgq_oracle.n_anchors(s)
        assert kgq.num_relations(s) == synth.N_RELS[s] == O.kgq_oracle.n_relations(s)
        assert kgq.num_branches(s) == O.kgq_oracle.n_branches(s)
        assert kgq.uses_negation(s) == O.kgq_oracle.uses_negation(s)
    assert kgq._lib.kgq_num_anchors(len(O.STRUCTURES)) == -1 and kgq._lib.kgq_num_anchors(-1) == -1
    with pytest.raises(kgq.KgqError, match="valid: 1p"):
        kgq.structure_id("4p")
    assert kgq.embedding_width("gqe", 400) == 400
    assert kgq.embedding_width("q2b", 400) == 800
    assert kgq.embedding_width("betae", 400) == 800


@pytest.mark.parametrize("n,w", [(1, 1), (7, 3), (14505, 8), (2_000_000, 8), (30, 4)])
def test_shard_range_matches_oracle(n, w):
    for r in range(w):
        assert kgq.shard_range(n, w, r) == O.shard_range(n, w, r)
    with pytest.raises(kgq.KgqError):
        kgq.shard_range(n, w, w)


def test_create_rejects_bad_config_without_crashing():
    cfg = kgq.KgqConfig(kgq.ABI_VERSION, 0, 100, 5, 30, 0, 0, 0.02, 0, 16, 10, 0, 1, 0)
    h = ctypes.c_void_p()
    st = kgq._lib.kgq_create(ctypes.byref(cfg), ctypes.byref(h))
    assert st == 1 and not h.value  # dim 30 is not a multiple of 4
    assert b"multiple of 4" in kgq._lib.kgq_last_error(None)
    cfg.dim = 32
    cfg.abi_version = 99
    assert kgq._lib.kgq_create(ctypes.byref(cfg), ctypes.byref(h)) == 1
    cfg.abi_version = kgq.ABI_VERSION
    cfg.max_k = 1000
    assert kgq._lib.kgq_create(ctypes.byref(cfg), ctypes.byref(h)) == 1
    kgq._lib.kgq_destroy(None)  # NULL-safe


def test_sass_is_sm100a():
    out = os.popen(f"cuobjdump -lelf {kgq.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_peer_entry_points_validate_without_a_gpu():
    """N2 host-side argument handling: NULL context, and the ShardedEngine merge switch."""
    assert kgq._lib.kgq_peer_bytes(None, 2) == -1
    assert kgq._lib.kgq_set_peers(None, 0, 2, None) == 1  # KGQ_EINVAL
    assert kgq._lib.kgq_merge_peers(None, 4, 5, None, None, None) == 1
    from paper_2503_02172_b200.sharded import ShardedEngine
    with pytest.raises(ValueError, match="merge"):
        ShardedEngine("betae", 100, 5, 8, merge="allreduce")
    with pytest.raises(ValueError, match="split"):
        ShardedEngine("betae", 100, 5, 8, split="rows")


@pytest.mark.parametrize("B,W", [(0, 1), (1, 8), (10, 3), (1024, 8), (1023, 8), (4096, 3), (7, 7)])
def test_query_range_partitions_the_batch(B, W):
    """Query-split mode (kgq_query_range): contiguous rows, ceil(B / W) per rank, the ranges
    tile [0, B) exactly in rank order."""
    c = -(-B // W) if B else 0
    got = [kgq.query_range(B, W, r) for r in range(W)]
    assert got[0][0] == 0 and got[-1][1] == B
    for r, (lo, hi) in enumerate(got):
        assert lo == min(B, r * c) and hi == min(B, lo + c)
        if r:
            assert lo == got[r - 1][1]
    with pytest.raises(kgq.KgqError):
        kgq.query_range(B, W, W)


def test_comm_entry_points_validate_without_a_gpu():
    """The communicator entry points' host-side checks (no device work)."""
    assert kgq._lib.kgq_comm_init(None, b"\0" * 128, 1, 0, 0) == 1       # NULL context
    assert kgq._lib.kgq_comm_destroy(None) == 1
    assert kgq._lib.kgq_rank_metrics(None, 1, None, None, None, None, None) == 1
    assert kgq._lib.kgq_nccl_unique_id(None) == 1
    assert kgq.STATUS[7] == "KGQ_ENCCL"
    uid = kgq.nccl_unique_id()   # NCCL's bootstrap id needs no GPU
    assert len(uid) == 128 and uid != kgq.nccl_unique_id()
