"""Thin Python binding of libkgq.so (include/kgq.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels behind the
C ABI.  PyTorch is used for device memory and stream handles.  There is no CPU fallback:
if libkgq.so is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# operand format of the tensor-core GEMMs: libkgq.so = fp16x2 (default), libkgq_bf16x3.so = the
# exact three-plane bf16 split (full fp32 range; KGQ_OPERANDS=bf16x3); KGQ_LIB_PATH: A/B builds only
OPERANDS = os.environ.get("KGQ_OPERANDS", "fp16x2")
LIB_PATH = os.environ.get("KGQ_LIB_PATH") or os.path.join(
    _HERE, "libkgq_bf16x3.so" if OPERANDS == "bf16x3" else "libkgq.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                      " (or `make -C paper_2503_02172_b200/csrc`)")
_lib = ctypes.CDLL(LIB_PATH)

ABI_VERSION = 1
MODELS = {"gqe": 0, "q2b": 1, "betae": 2}
STRUCTURES = ("1p", "2p", "3p", "2i", "3i", "pi", "ip", "2u", "up",
              "2in", "3in", "inp", "pin", "pni", "2u-DM", "up-DM")
STATUS = {0: "KGQ_OK", 1: "KGQ_EINVAL", 2: "KGQ_ERANGE", 3: "KGQ_EUNSUPPORTED",
          4: "KGQ_ESTATE", 5: "KGQ_ENOMEM", 6: "KGQ_ECUDA", 7: "KGQ_ENCCL"}
LAYER_PROJ_OUT, LAYER_PROJ_HIDDEN = 0, 1
LAYER_INTER_1, LAYER_INTER_2, LAYER_OFFSET_1, LAYER_OFFSET_2 = 16, 17, 18, 19
REL_MAIN, REL_OFFSET = 0, 1
STAGES = ("chain", "prep", "score", "topk", "dense")

# Every symbol include/kgq.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "kgq_create", "kgq_destroy", "kgq_last_error", "kgq_status_string", "kgq_num_anchors",
    "kgq_num_relations", "kgq_num_branches", "kgq_uses_negation", "kgq_structure_name",
    "kgq_structure_from_name", "kgq_embedding_width", "kgq_shard_range", "kgq_shard_begin",
    "kgq_shard_end", "kgq_load_entities", "kgq_load_relations", "kgq_load_linear",
    "kgq_finalize", "kgq_submit", "kgq_submit_host", "kgq_submit_host_async", "kgq_submit_mixed",
    "kgq_submit_mixed_host_async", "kgq_query_embedding", "kgq_merge_topk",
    "kgq_check_errors", "kgq_last_launch_count", "kgq_entity_terms", "kgq_profile_enable",
    "kgq_profile_read", "kgq_rank_answers", "kgq_peer_bytes", "kgq_set_peers", "kgq_merge_peers",
    "kgq_query_range", "kgq_nccl_unique_id", "kgq_comm_init", "kgq_comm_destroy", "kgq_rank_metrics",
    "kgq_ktime_enable", "kgq_ktime_read", "kgq_ktime_log", "kgq_set_option", "kgq_tensor_mmas_per_fma",
)
RANK_LOCAL, RANK_DIST, RANK_COUNT, RANK_FILTERED = 0, 1, 2, 3
SPLIT_ENTITIES, SPLIT_QUERIES = 0, 1


class KgqConfig(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_uint32), ("model", ctypes.c_int32),
                ("n_entity", ctypes.c_int64), ("n_relation", ctypes.c_int32),
                ("dim", ctypes.c_int32), ("hidden", ctypes.c_int32),
                ("n_hidden_layers", ctypes.c_int32), ("cen", ctypes.c_float),
                ("terminal", ctypes.c_int32), ("max_batch", ctypes.c_int32),
                ("max_k", ctypes.c_int32), ("device", ctypes.c_int32),
                ("world_size", ctypes.c_int32), ("rank", ctypes.c_int32)]


_P = ctypes.c_void_p
_I32, _I64 = ctypes.c_int32, ctypes.c_int64
_sig = {
    "kgq_create": (_I32, [ctypes.POINTER(KgqConfig), ctypes.POINTER(_P)]),
    "kgq_destroy": (None, [_P]),
    "kgq_last_error": (ctypes.c_char_p, [_P]),
    "kgq_status_string": (ctypes.c_char_p, [_I32]),
    "kgq_num_anchors": (_I32, [_I32]),
    "kgq_num_relations": (_I32, [_I32]),
    "kgq_num_branches": (_I32, [_I32]),
    "kgq_uses_negation": (_I32, [_I32]),
    "kgq_structure_name": (ctypes.c_char_p, [_I32]),
    "kgq_structure_from_name": (_I32, [ctypes.c_char_p]),
    "kgq_embedding_width": (_I32, [_I32, _I32]),
    "kgq_shard_range": (_I32, [_I64, _I32, _I32, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "kgq_shard_begin": (_I64, [_P]),
    "kgq_shard_end": (_I64, [_P]),
    "kgq_load_entities": (_I32, [_P, _P, _I64, _I64]),
    "kgq_load_relations": (_I32, [_P, _I32, _P, _I32]),
    "kgq_load_linear": (_I32, [_P, _I32, _P, _P, _I32, _I32]),
    "kgq_finalize": (_I32, [_P]),
    "kgq_submit": (_I32, [_P, _I32, _I32, _P, _P, _I32, _P, _P, _P, _P]),
    "kgq_submit_host": (_I32, [_P, _I32, _I32, _P, _P, _I32, _P, _P, _P]),
    "kgq_submit_host_async": (_I32, [_P, _I32, _I32, _P, _P, _I32, _P, _P, _P]),
    "kgq_submit_mixed": (_I32, [_P, _I32, _P, _P, _P, _P, _I32, _P, _P, _P]),
    "kgq_submit_mixed_host_async": (_I32, [_P, _I32, _P, _P, _P, _P, _I32, _P, _P, _P]),
    "kgq_query_embedding": (_I32, [_P, _I32, _I32, _P, _P, _P, _P]),
    "kgq_merge_topk": (_I32, [_P, _I32, _I32, _I32, _P, _P, _P, _P, _P]),
    "kgq_check_errors": (_I32, [_P, _P]),
    "kgq_last_launch_count": (_I32, [_P]),
    "kgq_entity_terms": (_I32, [_P, _P, _P]),
    "kgq_profile_enable": (_I32, [_P, _I32]),
    "kgq_rank_answers": (_I32, [_P, _I32, _I32, _P, _P, _P, _P, _I32, _I32, _P, _P, _P]),
    "kgq_peer_bytes": (_I64, [_P, _I32]),
    "kgq_set_peers": (_I32, [_P, _I32, _I32, ctypes.POINTER(_P)]),
    "kgq_merge_peers": (_I32, [_P, _I32, _I32, _P, _P, _P]),
    "kgq_profile_read": (_I32, [_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64),
                              ctypes.POINTER(ctypes.c_double)]),
    "kgq_query_range": (_I32, [_I32, _I32, _I32, ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "kgq_nccl_unique_id": (_I32, [ctypes.c_char_p]),
    "kgq_comm_init": (_I32, [_P, ctypes.c_char_p, _I32, _I32, _I32]),
    "kgq_comm_destroy": (_I32, [_P]),
    "kgq_rank_metrics": (_I32, [_P, _I32, _P, _P, _P, _P, _P]),
    "kgq_ktime_enable": (_I32, [_P, _I32]),
    "kgq_ktime_read": (_I32, [_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64)]),
    "kgq_ktime_log": (_I64, [_P, _P, _I64]),
    "kgq_set_option": (_I32, [_P, _I32, _I64]),
    "kgq_tensor_mmas_per_fma": (_I32, []),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class KgqError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = STATUS.get(status, status)


def tensor_mmas_per_fma() -> int:
    """MMAs per useful fp32 multiply-add of this build's GEMMs (3: fp16x2, 6: bf16x3)."""
    return int(_lib.kgq_tensor_mmas_per_fma())


def structure_id(s) -> int:
    if isinstance(s, (int, np.integer)):
        return int(s)
    v = _lib.kgq_structure_from_name(str(s).encode())
    if v < 0:
        raise KgqError(1, f"unknown structure {s!r}; valid: {', '.join(STRUCTURES)}")
    return v


def num_anchors(s): return _lib.kgq_num_anchors(structure_id(s))
def num_relations(s): return _lib.kgq_num_relations(structure_id(s))
def num_branches(s): return _lib.kgq_num_branches(structure_id(s))
def uses_negation(s): return bool(_lib.kgq_uses_negation(structure_id(s)))
def embedding_width(model, dim): return _lib.kgq_embedding_width(MODELS[model], dim)


def shard_range(n_entity, world_size, rank):
    b, e = _I64(), _I64()
    st = _lib.kgq_shard_range(n_entity, world_size, rank, ctypes.byref(b), ctypes.byref(e))
    if st:
        raise KgqError(st, "bad shard arguments")
    return b.value, e.value


def query_range(batch, world_size, rank):
    """Rows [lo, hi) of a replicated batch that `rank` runs in query-split mode (kgq_query_range)."""
    lo, hi = _I32(), _I32()
    st = _lib.kgq_query_range(batch, world_size, rank, ctypes.byref(lo), ctypes.byref(hi))
    if st:
        raise KgqError(st, _lib.kgq_last_error(None).decode())
    return lo.value, hi.value


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (kgq_nccl_unique_id); raises KgqError(KGQ_ENCCL) without NCCL."""
    import torch  # noqa: F401  -- load the process's NCCL (torch's) before libkgq looks for one
    buf = ctypes.create_string_buffer(128)
    st = _lib.kgq_nccl_unique_id(buf)
    if st:
        raise KgqError(st, _lib.kgq_last_error(None).decode())
    return buf.raw


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _on_stream(stream):
    """Context that makes `stream` current for the binding's own allocations and staging
    copies (so the caching allocator and the copies are ordered with the library's launches on
    that stream), after making it wait for the caller's current stream (which produced the
    inputs).  No-op for stream=None (the library then runs on the current stream)."""
    import contextlib
    import torch
    if stream is None:
        return contextlib.nullcontext()
    cur = torch.cuda.current_stream()
    if stream != cur:
        stream.wait_stream(cur)
    return torch.cuda.stream(stream)


def layer_id(name: str) -> int:
    """synth / nn.Module parameter name -> KGQ_LAYER_* id."""
    if name == "proj.layer0":
        return LAYER_PROJ_OUT
    if name.startswith("proj.layer"):
        return LAYER_PROJ_HIDDEN + int(name[len("proj.layer"):]) - 1
    return {"inter.layer1": LAYER_INTER_1, "inter.layer2": LAYER_INTER_2,
            "offset.layer1": LAYER_OFFSET_1, "offset.layer2": LAYER_OFFSET_2}[name]


class Engine:
    """One libkgq context: one model, one entity shard, one device."""

    def __init__(self, model, n_entity, n_relation, dim, *, hidden=1600, n_hidden_layers=2,
                 cen=0.02, terminal="regularizer", max_batch=1024, max_k=16, device=0,
                 world_size=1, rank=0):
        self.model = model
        self.dim = dim
        cfg = KgqConfig(ABI_VERSION, MODELS[model], n_entity, n_relation, dim, hidden,
                        n_hidden_layers, cen, 0 if terminal == "regularizer" else 1, max_batch,
                        max_k, device, world_size, rank)
        h = _P()
        st = _lib.kgq_create(ctypes.byref(cfg), ctypes.byref(h))
        if st:
            raise KgqError(st, _lib.kgq_last_error(None).decode())
        self._h = h
        self.cfg = cfg
        self.device = device
        self.shard = (_lib.kgq_shard_begin(h), _lib.kgq_shard_end(h))
        self.width = embedding_width(model, dim)

    def close(self):
        if getattr(self, "_h", None):
            _lib.kgq_destroy(self._h)
            self._h = None

    __del__ = close

    def _check(self, st):
        if st:
            raise KgqError(st, _lib.kgq_last_error(self._h).decode())

    # ---- tables ---------------------------------------------------------------------------
    def load_entities(self, rows: np.ndarray, first_row: int = 0):
        rows = np.ascontiguousarray(rows, dtype=np.float32)
        self._check(_lib.kgq_load_entities(self._h, rows.ctypes.data, first_row, rows.shape[0]))

    def load_relations(self, rows: np.ndarray, which: int = REL_MAIN):
        rows = np.ascontiguousarray(rows, dtype=np.float32)
        self._check(_lib.kgq_load_relations(self._h, which, rows.ctypes.data, rows.shape[0]))

    def load_linear(self, name_or_id, W: np.ndarray, b: np.ndarray):
        lid = layer_id(name_or_id) if isinstance(name_or_id, str) else int(name_or_id)
        W = np.ascontiguousarray(W, dtype=np.float32)
        b = np.ascontiguousarray(b, dtype=np.float32)
        self._check(_lib.kgq_load_linear(self._h, lid, W.ctypes.data, b.ctypes.data, W.shape[0],
                                         W.shape[1]))

    def load_tables(self, t: dict, finalize: bool = True):
        """Load a synth-format table dict ('entity', 'relation', 'offset', 'W:*', 'b:*')."""
        ent = t["entity"]
        step = 1 << 18
        for r0 in range(0, ent.shape[0], step):
            self.load_entities(ent[r0:r0 + step], r0)
        self.load_relations(t["relation"], REL_MAIN)
        if self.model == "q2b":
            self.load_relations(t["offset"], REL_OFFSET)
        for k in t:
            if k.startswith("W:"):
                self.load_linear(k[2:], t[k], t["b:" + k[2:]])
        if finalize:
            self.finalize()

    def finalize(self):
        self._check(_lib.kgq_finalize(self._h))

    # ---- hot path -------------------------------------------------------------------------
    def submit(self, structure, anchors, rels, k, *, out=None, shard_dist=False, stream=None):
        """anchors/rels: int32 CUDA tensors [B, n_a] / [B, n_r].  Returns (dist [B,k],
        ids [B,k]) CUDA tensors (and the [B, shard] distance matrix if shard_dist)."""
        import torch
        s = structure_id(structure)
        B = anchors.shape[0]
        dev = anchors.device
        with _on_stream(stream):
            if out is None:
                td = torch.empty((B, k), dtype=torch.float32, device=dev)
                ti = torch.empty((B, k), dtype=torch.int32, device=dev)
            else:
                td, ti = out
            sd = (torch.empty((B, self.shard[1] - self.shard[0]), dtype=torch.float32, device=dev)
                  if shard_dist else None)
        self._check(_lib.kgq_submit(self._h, s, B, _ptr(anchors), _ptr(rels), k, _ptr(td),
                                    _ptr(ti), _ptr(sd), _stream(stream)))
        return (td, ti, sd) if shard_dist else (td, ti)

    def submit_mixed(self, groups, k, *, out=None, stream=None):
        """Mixed-structure batch (kgq_submit_mixed): groups = [(structure, anchors, rels), ...]
        with int32 CUDA tensors [B_i, n_a] / [B_i, n_r].  Returns (dist, ids) CUDA tensors
        [sum B_i, k], rows in group order."""
        import torch
        ss = (ctypes.c_int32 * len(groups))(*[structure_id(g[0]) for g in groups])
        bs = (ctypes.c_int32 * len(groups))(*[int(g[1].shape[0]) for g in groups])
        dev = groups[0][1].device if groups else torch.device("cuda")
        # inputs packed into per-engine staging buffers (stable addresses: an identical later call
        # replays the library's captured graph of the whole mixed submit)
        na = sum(int(g[1].numel()) for g in groups)
        nr = sum(int(g[2].numel()) for g in groups)
        Q = sum(int(g[1].shape[0]) for g in groups)
        with _on_stream(stream):
            st = getattr(self, "_mix_in", None)
            if st is None or st[0].numel() < na or st[1].numel() < nr or st[0].device != dev:
                st = (torch.empty(max(na, 1), dtype=torch.int32, device=dev),
                      torch.empty(max(nr, 1), dtype=torch.int32, device=dev))
                self._mix_in = st
                self._mix_ev = None
            a, r = st[0][:na], st[1][:nr]
            # the staging buffers are reused: the previous mixed submit (possibly on another
            # stream) must have read them before they are overwritten
            if getattr(self, "_mix_ev", None) is not None:
                torch.cuda.current_stream().wait_event(self._mix_ev)
            if groups:
                torch.cat([g[1].reshape(-1).to(torch.int32) for g in groups], out=a)
                torch.cat([g[2].reshape(-1).to(torch.int32) for g in groups], out=r)
            if out is None:
                td = torch.empty((Q, k), dtype=torch.float32, device=dev)
                ti = torch.empty((Q, k), dtype=torch.int32, device=dev)
            else:
                td, ti = out
            self._keep = (a, r)  # the launch is asynchronous: keep the concatenated inputs alive
            self._check(_lib.kgq_submit_mixed(self._h, len(groups), ss, bs, _ptr(a), _ptr(r), k, _ptr(td),
                                              _ptr(ti), _stream(stream)))
            if groups:
                self._mix_ev = torch.cuda.Event()
                self._mix_ev.record()
        return td, ti

    def submit_mixed_packed(self, structures, batches, anchors, rels, k, out, stream=None):
        """kgq_submit_mixed on inputs already packed in group order (int32 CUDA tensors: the groups'
        [B_i, n_a] anchor blocks back to back, likewise the relations) -- no staging copy, so a
        repeated call with the same tensors replays the library's captured graph as is."""
        ss = (ctypes.c_int32 * len(structures))(*[structure_id(s) for s in structures])
        bs = (ctypes.c_int32 * len(batches))(*[int(b) for b in batches])
        td, ti = out
        self._check(_lib.kgq_submit_mixed(self._h, len(structures), ss, bs, _ptr(anchors), _ptr(rels), k,
                                          _ptr(td), _ptr(ti), _stream(stream)))
        return td, ti

    def submit_mixed_host(self, structures, batches, anchors: np.ndarray, rels: np.ndarray, k: int, out,
                          stream=None):
        """kgq_submit_mixed_host_async: host int32 inputs packed in group order (pinned for
        overlap), host outputs out = (dist [Q, k] fp32, ids [Q, k] int32); asynchronous -- valid
        after `stream` is synchronised."""
        ss = (ctypes.c_int32 * len(structures))(*[structure_id(s) for s in structures])
        bs = (ctypes.c_int32 * len(batches))(*[int(b) for b in batches])
        td, ti = out
        self._check(_lib.kgq_submit_mixed_host_async(self._h, len(structures), ss, bs, anchors.ctypes.data,
                                                     rels.ctypes.data, k, td.ctypes.data, ti.ctypes.data,
                                                     _stream(stream)))
        return td, ti

    def submit_host(self, structure, anchors: np.ndarray, rels: np.ndarray, k: int,
                    out=None, stream=None, sync=True):
        """End-to-end call with host buffers (H2D + path + D2H inside the library).  sync=False
        (kgq_submit_host_async): returns after enqueueing; the outputs are valid after the
        stream is synchronised (use pinned buffers for overlap)."""
        s = structure_id(structure)
        anchors = np.ascontiguousarray(anchors, dtype=np.int32)
        rels = np.ascontiguousarray(rels, dtype=np.int32)
        B = anchors.shape[0]
        if out is None:
            td = np.empty((B, k), np.float32)
            ti = np.empty((B, k), np.int32)
        else:
            td, ti = out
        fn = _lib.kgq_submit_host if sync else _lib.kgq_submit_host_async
        self._check(fn(self._h, s, B, anchors.ctypes.data, rels.ctypes.data, k,
                       td.ctypes.data, ti.ctypes.data, _stream(stream)))
        return td, ti

    def query_embedding(self, structure, anchors, rels, stream=None):
        import torch
        s = structure_id(structure)
        B = anchors.shape[0]
        with _on_stream(stream):
            out = torch.empty((B, num_branches(s), self.width), dtype=torch.float32,
                              device=anchors.device)
        self._check(_lib.kgq_query_embedding(self._h, s, B, _ptr(anchors), _ptr(rels), _ptr(out),
                                             _stream(stream)))
        return out

    def merge_topk(self, parts_dist, parts_id, k, stream=None):
        """parts_*: CUDA tensors [W, B, k] -> (dist [B,k], ids [B,k])."""
        import torch
        W, B, kk = parts_dist.shape
        with _on_stream(stream):
            od = torch.empty((B, k), dtype=torch.float32, device=parts_dist.device)
            oi = torch.empty((B, k), dtype=torch.int32, device=parts_dist.device)
            pd, pi = parts_dist.contiguous(), parts_id.contiguous()
            self._check(_lib.kgq_merge_topk(self._h, W, B, kk, _ptr(pd), _ptr(pi), _ptr(od), _ptr(oi),
                                            _stream(stream)))
        return od, oi

    # ---- N2: fused top-k all-gather over peer memory (kgq_set_peers / kgq_merge_peers) ----
    def peer_bytes(self, world):
        """Size in bytes of this context's per-rank peer buffer for `world` ranks."""
        n = int(_lib.kgq_peer_bytes(self._h, world))
        if n < 0:
            raise KgqError(-1, f"kgq_peer_bytes: bad world {world}")
        return n

    def set_peers(self, rank, world, ptrs):
        """Registers every rank's peer buffer (device addresses, this context = rank); world 0
        turns the push off."""
        arr = (ctypes.c_void_p * max(1, len(ptrs)))(*[int(p) for p in ptrs])
        self._check(_lib.kgq_set_peers(self._h, rank, world, arr if world else None))

    def merge_peers(self, batch, k, out=None, stream=None):
        """Waits for every rank's push of the current submit and merges: (dist, ids) [batch, k]."""
        import torch
        with _on_stream(stream):
            if out is None:
                td = torch.empty((batch, k), dtype=torch.float32, device=f"cuda:{self.device}")
                ti = torch.empty((batch, k), dtype=torch.int32, device=f"cuda:{self.device}")
            else:
                td, ti = out
        self._check(_lib.kgq_merge_peers(self._h, batch, k, _ptr(td), _ptr(ti), _stream(stream)))
        return td, ti

    # ---- multi-GPU data plane: the library's NCCL communicator (kgq_comm_init) ----------------
    def comm_init(self, unique_id: bytes, world, rank, split=SPLIT_ENTITIES):
        """Collective over the job's `world` ranks (one context each, same unique_id)."""
        import torch  # noqa: F401  -- the process's NCCL (torch's) is the one libkgq binds to
        if len(unique_id) != 128:
            raise ValueError("the NCCL unique id is 128 bytes")
        self._check(_lib.kgq_comm_init(self._h, unique_id, world, rank, split))

    def comm_destroy(self):
        self._check(_lib.kgq_comm_destroy(self._h))

    def rank_metrics(self, ans_off, ranks, hard=None, stream=None):
        """MRR, Hits@1/3/10 and the number of queries averaged (kgq_rank_metrics): fp64 CUDA
        tensor [5].  ranks: int32 1-based filtered ranks in the CSR layout of ans_off."""
        import torch
        B = int(ans_off.shape[0]) - 1
        with _on_stream(stream):
            out = torch.empty(5, dtype=torch.float64, device=ranks.device)
        self._check(_lib.kgq_rank_metrics(self._h, B, _ptr(ans_off), _ptr(ranks), _ptr(hard), _ptr(out),
                                          _stream(stream)))
        return out

    def rank_answers(self, structure, anchors, rels, ans_off, ans_id, mode=RANK_LOCAL,
                     ans_dist=None, stream=None):
        """N1 filtered ranking (kgq_rank_answers).  ans_off int32 [B+1], ans_id int32 [n] CUDA
        tensors (CSR of each query's easy + hard answers).  Returns (ans_dist, count): the
        filtered rank of answer j is 1 + count[j] (summed over shards); with RANK_FILTERED
        `count` already holds that rank (over all shards through the communicator)."""
        import torch
        s = structure_id(structure)
        B = anchors.shape[0]
        n = int(ans_id.shape[0])
        with _on_stream(stream):
            if ans_dist is None:
                ans_dist = torch.empty(n, dtype=torch.float32, device=anchors.device)
            count = torch.zeros(n, dtype=torch.int32, device=anchors.device)
        self._check(_lib.kgq_rank_answers(self._h, s, B, _ptr(anchors), _ptr(rels), _ptr(ans_off),
                                          _ptr(ans_id), n, mode, _ptr(ans_dist),
                                          _ptr(count) if mode != RANK_DIST else None,
                                          _stream(stream)))
        return ans_dist, count

    def check_errors(self, stream=None):
        self._check(_lib.kgq_check_errors(self._h, _stream(stream)))

    def last_launch_count(self) -> int:
        return _lib.kgq_last_launch_count(self._h)

    def entity_terms(self, stream=None):
        import torch
        ns = self.shard[1] - self.shard[0]
        out = torch.empty((3, self.dim, ns), dtype=torch.float32, device=f"cuda:{self.device}")
        self._check(_lib.kgq_entity_terms(self._h, _ptr(out), _stream(stream)))
        return out

    def set_fused_topk(self, mode: str):
        """kgq_set_option(KGQ_OPT_FUSED_TOPK): "off" (write the distance block), "on" (fuse the top-k
        into the BetaE tensor-core scorer whenever eligible), "auto" (default)."""
        self._check(_lib.kgq_set_option(self._h, 1, {"off": 0, "on": 1, "auto": 2}[mode]))

    def ktime(self, on: bool = True):
        """In-kernel launch spans of the tcgen05 GEMM (kgq_ktime_enable)."""
        self._check(_lib.kgq_ktime_enable(self._h, 1 if on else 0))

    def ktime_read(self):
        """{"dense": (ms, launches), "score": (ms, launches)} since the last read."""
        ms = (ctypes.c_double * 2)()
        n = (_I64 * 2)()
        self._check(_lib.kgq_ktime_read(self._h, ms, n))
        return {"dense": (ms[0], n[0]), "score": (ms[1], n[1])}

    def ktime_log(self, cap=1 << 16):
        """numpy uint64 [n, 3] of GEMM launch spans {start ns, end ns, stage 0 dense / 1 score}."""
        buf = np.zeros((cap, 3), np.uint64)
        n = int(_lib.kgq_ktime_log(self._h, buf.ctypes.data, cap))
        if n < 0:
            raise KgqError(6, "kgq_ktime_log failed")
        return buf[:min(n, cap)].copy()

    def profile(self, on: bool = True):
        self._check(_lib.kgq_profile_enable(self._h, 1 if on else 0))

    def profile_read(self):
        """{stage: (device ms, timed regions, algorithmic work)} since the last read."""
        k = len(STAGES)
        ms = (ctypes.c_double * k)()
        n = (_I64 * k)()
        w = (ctypes.c_double * k)()
        self._check(_lib.kgq_profile_read(self._h, ms, n, w))
        return {STAGES[i]: (ms[i], n[i], w[i]) for i in range(k)}
