"""Multi-GPU front end: one process per GPU, torch.distributed only to start
the job and to hand the NCCL unique id around; the data plane runs inside libkgq.so.

Two splits of the replicated query batch, both behind kgq_comm_init (include/kgq.h):
  split="entities" (north_star; the 2M-entity table): rank r owns the contiguous entity range
      kgq_shard_range(N, W, r), scores it and selects its local top-k; the library's own NCCL
      communicator all-gathers the W [B, k] lists and its merge kernel (a9) writes the global
      top-k on every rank -- all inside one kgq_submit, on the caller's stream.
  split="queries" (small tables such as FB15k-237, where the operator chain dominates the step):
      every rank holds the whole table and runs only its rows kgq_query_range(B, W, r) of the
      batch; one all-gather inside kgq_submit returns the whole batch's top-k on every rank.

merge (entities only):
  "nccl"  the library's communicator (default; falls back to "torch" -- on every rank alike --
          if NCCL cannot be loaded, saying why in `merge_mode`);
  "p2p"   N2: the all-gather fused into the top-k kernel over symmetric peer memory
          (kgq_set_peers / kgq_merge_peers), no NCCL on the data path;
  "torch" torch.distributed all-gather + kgq_merge_topk: the host-composed baseline (and the
          path the gloo CPU tests exercise).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .kgq import (RANK_COUNT, RANK_DIST, RANK_FILTERED, RANK_LOCAL, SPLIT_ENTITIES, SPLIT_QUERIES,
                  Engine, KgqError, nccl_unique_id)


def all_gather_topk(td: torch.Tensor, ti: torch.Tensor, group=None):
    """[B, k] local (dist, id) on every rank -> ([W, B, k], [W, B, k]) in rank order
    (torch.distributed; the merge="torch" path)."""
    W = dist.get_world_size(group)
    B = td.shape[0]
    gd = torch.empty((W * B,) + tuple(td.shape[1:]), dtype=td.dtype, device=td.device)
    gi = torch.empty((W * B,) + tuple(ti.shape[1:]), dtype=ti.dtype, device=ti.device)
    dist.all_gather_into_tensor(gd, td.contiguous(), group=group)
    dist.all_gather_into_tensor(gi, ti.contiguous(), group=group)
    return gd.view((W,) + tuple(td.shape)), gi.view((W,) + tuple(ti.shape))


def _device_of_group(group, dev):
    return "cpu" if dist.get_backend(group) == "gloo" else torch.device("cuda", dev)


class ShardedEngine:
    """This rank's part of a W-way split model (see the module docstring)."""

    def __init__(self, model, n_entity, n_relation, dim, *, split="entities", group=None, device=None,
                 merge="nccl", **kw):
        if split not in ("entities", "queries"):
            raise ValueError(f"split must be 'entities' or 'queries', not {split!r}")
        if merge not in ("nccl", "p2p", "torch"):
            raise ValueError(f"merge must be 'nccl', 'p2p' or 'torch', not {merge!r}")
        if split == "queries" and merge != "nccl":
            raise ValueError("split='queries' runs through the library's communicator (merge='nccl')")
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.split = split
        dev = torch.cuda.current_device() if device is None else device
        self.dev = dev
        shard_w, shard_r = (self.world, self.rank) if split == "entities" else (1, 0)
        self.engine = Engine(model, n_entity, n_relation, dim, device=dev, world_size=shard_w, rank=shard_r, **kw)
        self.shard = self.engine.shard
        self.merge_mode = "local" if self.world == 1 else merge
        self.p2p_check = True  # N2: raise right after a merge whose device error word is set
        self._peer_buf = None
        self._launches = 0
        if self.world > 1 and merge == "nccl":
            why = self._setup_comm()
            if why is not None:
                if split == "queries":
                    raise KgqError(7, f"query split needs the library communicator: {why}")
                self.merge_mode = f"torch (library communicator unavailable: {why})"
        elif self.world > 1 and merge == "p2p":
            why = self._setup_p2p(dev)
            if why is not None:  # no symmetric memory here: the torch merge gives the same result
                self.merge_mode = f"torch (p2p unavailable: {why})"

    # ---- setup ------------------------------------------------------------------------------
    def _agree(self, ok: bool) -> bool:
        """Collective AND of a per-rank success flag: every rank takes the same branch (a rank
        that failed a setup step must not skip a collective the others enter)."""
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=_device_of_group(self.group, self.dev))
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return bool(t.item())

    def _setup_comm(self):
        """Rank 0 draws the NCCL unique id (kgq_nccl_unique_id) and broadcasts it; every rank
        then creates the library communicator (kgq_comm_init).  None on success, else why (the
        same decision on every rank)."""
        uid, why = None, None
        if self.rank == 0:
            try:
                uid = nccl_unique_id()
            except KgqError as e:
                why = str(e)
        box = [uid if why is None else None, why]
        src = dist.get_global_rank(self.group, 0) if self.group is not None else 0
        dist.broadcast_object_list(box, src=src, group=self.group)
        uid, why = box
        if uid is None:
            return why or "no NCCL unique id"
        try:  # collective: every rank got here with the same id
            self.engine.comm_init(uid, self.world, self.rank,
                                  SPLIT_ENTITIES if self.split == "entities" else SPLIT_QUERIES)
        except KgqError as e:
            why = str(e)
        return None if self._agree(why is None) else (why or "kgq_comm_init failed on another rank")

    def _setup_p2p(self, dev):
        """Symmetric peer buffers for N2, set up step by step with a collective agreement after
        every step that can fail on one rank only; returns None on success, else the first
        failure's text (the same decision on every rank)."""
        why, buf, h = None, None, None
        try:
            import torch.distributed._symmetric_memory as symm_mem
            buf = symm_mem.empty(self.engine.peer_bytes(self.world), dtype=torch.uint8,
                                 device=torch.device("cuda", dev))
        except Exception as e:
            why = f"allocation: {type(e).__name__}: {e}"
        if not self._agree(why is None):
            return why or "allocation failed on another rank"
        try:  # collective on every rank (all of them got here)
            h = symm_mem.rendezvous(buf, self.group if self.group is not None else dist.group.WORLD)
            ptrs = list(h.buffer_ptrs)
            if len(ptrs) != self.world:
                raise RuntimeError(f"symmetric memory returned {len(ptrs)} buffers for {self.world} ranks")
            self.engine.set_peers(self.rank, self.world, ptrs)
        except Exception as e:
            why = f"rendezvous: {type(e).__name__}: {e}"
        if not self._agree(why is None):
            if why is None:
                self.engine.set_peers(self.rank, 0, [])  # another rank failed: push off here too
            return why or "rendezvous failed on another rank"
        dist.barrier(group=self.group)  # every rank's buffer is reset before anyone pushes
        self._peer_buf = (buf, h)
        return None

    def load_tables(self, t, finalize=True):
        self.engine.load_tables(t, finalize)

    # ---- hot path ---------------------------------------------------------------------------
    def _merge_p2p(self, batch, k, stream):
        out = self.engine.merge_peers(batch, k, stream=stream)
        if self.p2p_check:
            # a timed-out merge poisons the peer session on every rank (peer.cuh): raise here
            # instead of returning its NaN / -1 rows; recovery = set_peers on every rank
            self.engine.check_errors(stream)
        return out

    def _finish(self, td, ti, k, stream):
        self._launches = self.engine.last_launch_count()
        if self.merge_mode.startswith("p2p"):
            self._launches += 1
            return self._merge_p2p(td.shape[0], k, stream)
        if self.merge_mode.startswith("torch"):
            self._launches += 1  # the merge kernel (NCCL's own kernels are not counted)
            gd, gi = all_gather_topk(td, ti, self.group)
            return self.engine.merge_topk(gd, gi, k, stream=stream)
        return td, ti  # "local" or "nccl": the library returned the global result

    def submit(self, structure, anchors, rels, k, stream=None):
        """Global top-k of the replicated batch (every rank passes the same anchors / rels)."""
        td, ti = self.engine.submit(structure, anchors, rels, k, stream=stream)
        return self._finish(td, ti, k, stream)

    def submit_mixed(self, groups, k, stream=None):
        """Mixed-structure batch (kgq_submit_mixed) -> global top-k [sum B_i, k]."""
        td, ti = self.engine.submit_mixed(groups, k, stream=stream)
        return self._finish(td, ti, k, stream)

    def submit_mixed_packed(self, structures, batches, anchors, rels, k, out, stream=None):
        """kgq_submit_mixed on inputs packed in group order (Engine.submit_mixed_packed) -> global
        top-k.  With the library communicator (merge "nccl") `out` receives the global result."""
        td, ti = self.engine.submit_mixed_packed(structures, batches, anchors, rels, k, out, stream=stream)
        return self._finish(td, ti, k, stream)

    def submit_mixed_host(self, structures, batches, anchors, rels, k, out, stream=None):
        """kgq_submit_mixed_host_async (host buffers, asynchronous): only where the library returns
        the global result itself (one rank, or its communicator)."""
        if self.merge_mode not in ("local", "nccl"):
            raise KgqError(4, f"host-buffer mixed submit needs the library communicator (merge {self.merge_mode})")
        self.engine.submit_mixed_host(structures, batches, anchors, rels, k, out, stream=stream)
        self._launches = self.engine.last_launch_count()
        return out

    def last_launch_count(self):
        return self._launches

    def rank_answers(self, structure, anchors, rels, ans_off, ans_id, stream=None):
        """N1 filtered ranks (1-based) of every answer across all shards (kgq_rank_answers)."""
        if self.world == 1 or self.split == "queries" or self.merge_mode == "nccl":
            # one table, or the library's communicator reduces over the shards inside
            return self.engine.rank_answers(structure, anchors, rels, ans_off, ans_id, RANK_FILTERED,
                                            stream=stream)[1]
        ad, _ = self.engine.rank_answers(structure, anchors, rels, ans_off, ans_id, RANK_DIST, stream=stream)
        dist.all_reduce(ad, op=dist.ReduceOp.MIN, group=self.group)
        _, cnt = self.engine.rank_answers(structure, anchors, rels, ans_off, ans_id, RANK_COUNT, ans_dist=ad,
                                          stream=stream)
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=self.group)
        return cnt + 1

    def metrics(self, ans_off, ranks, hard=None, stream=None):
        """MRR / Hits@1,3,10 over the batch (kgq_rank_metrics): dict of floats."""
        m = self.engine.rank_metrics(ans_off, ranks, hard, stream=stream).cpu().tolist()
        return dict(zip(("mrr", "hits1", "hits3", "hits10", "queries"), m))


def answers_csr(answer_lists):
    """[array of global ids per query] -> (ans_off int32 [B+1], ans_id int32 [n]) numpy."""
    import numpy as np
    off = np.zeros(len(answer_lists) + 1, np.int32)
    off[1:] = np.cumsum([len(a) for a in answer_lists])
    ids = np.concatenate([np.asarray(a, np.int32) for a in answer_lists]) if answer_lists else np.zeros(0, np.int32)
    return off, ids.astype(np.int32)


__all__ = ["ShardedEngine", "all_gather_topk", "answers_csr", "RANK_LOCAL"]
