"""Entity-sharded multi-GPU path: one process per GPU, torch.distributed for
the plumbing.

Rank r owns the contiguous entity range kgq_shard_range(N, W, r); queries are replicated;
each rank scores its shard and selects its local top-k (global ids) on its GPU; one
all-gather of the W x [B, k] (distance, id) pairs exchanges them (NCCL over NVLink on the
GPU box, gloo in the CPU tests); kgq_merge_topk merges W*k -> k on every rank.

merge="p2p" (N2): the all-gather is fused into the top-k kernel instead -- each
rank's top-k writes its rows straight into every rank's symmetric-memory peer buffer over
NVLink and releases a per-row flag; kgq_merge_peers waits for the flags on the device and
merges (no NCCL call, no host synchronisation on the data path).  The buffers come from
torch's symmetric memory (torch.distributed._symmetric_memory); if it is unavailable the
engine falls back to merge="nccl" and says so in `merge_mode`.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .kgq import RANK_COUNT, RANK_DIST, RANK_LOCAL, Engine


def all_gather_topk(td: torch.Tensor, ti: torch.Tensor, group=None):
    """[B, k] local (dist, id) on every rank -> ([W, B, k], [W, B, k]) in rank order."""
    W = dist.get_world_size(group)
    B = td.shape[0]
    gd = torch.empty((W * B,) + tuple(td.shape[1:]), dtype=td.dtype, device=td.device)
    gi = torch.empty((W * B,) + tuple(ti.shape[1:]), dtype=ti.dtype, device=ti.device)
    dist.all_gather_into_tensor(gd, td.contiguous(), group=group)
    dist.all_gather_into_tensor(gi, ti.contiguous(), group=group)
    return gd.view((W,) + tuple(td.shape)), gi.view((W,) + tuple(ti.shape))


class ShardedEngine:
    """This rank's shard of a W-way entity-sharded model."""

    def __init__(self, model, n_entity, n_relation, dim, *, group=None, device=None, merge="nccl", **kw):
        if merge not in ("nccl", "p2p"):
            raise ValueError(f"merge must be 'nccl' or 'p2p', not {merge!r}")
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        dev = torch.cuda.current_device() if device is None else device
        self.engine = Engine(model, n_entity, n_relation, dim, device=dev,
                             world_size=self.world, rank=self.rank, **kw)
        self.shard = self.engine.shard
        self.merge_mode = "nccl"
        self._peer_buf = None
        self._launches = 0
        if merge == "p2p" and self.world > 1:
            try:
                self._setup_p2p(dev)
                self.merge_mode = "p2p"
            except Exception as e:  # no symmetric memory here: the NCCL merge gives the same result
                self.merge_mode = f"nccl (p2p unavailable: {type(e).__name__}: {e})"

    def _setup_p2p(self, dev):
        import torch.distributed._symmetric_memory as symm_mem
        n = self.engine.peer_bytes(self.world)
        buf = symm_mem.empty(n, dtype=torch.uint8, device=torch.device("cuda", dev))
        h = symm_mem.rendezvous(buf, self.group if self.group is not None else dist.group.WORLD)
        ptrs = list(h.buffer_ptrs)
        if len(ptrs) != self.world:
            raise RuntimeError(f"symmetric memory returned {len(ptrs)} buffers for {self.world} ranks")
        self.engine.set_peers(self.rank, self.world, ptrs)
        dist.barrier(group=self.group)  # every rank's buffer is reset before anyone pushes
        self._peer_buf = (buf, h)

    def load_tables(self, t, finalize=True):
        self.engine.load_tables(t, finalize)

    def submit(self, structure, anchors, rels, k, stream=None):
        """Global top-k of the replicated batch: local top-k -> all-gather -> merge."""
        td, ti = self.engine.submit(structure, anchors, rels, k, stream=stream)
        self._launches = self.engine.last_launch_count()
        if self.world == 1:
            return td, ti
        self._launches += 1  # the merge kernel (NCCL's own kernels are not counted)
        if self.merge_mode == "p2p":
            return self.engine.merge_peers(td.shape[0], k, stream=stream)
        gd, gi = all_gather_topk(td, ti, self.group)
        return self.engine.merge_topk(gd, gi, k, stream=stream)

    def submit_mixed(self, groups, k, stream=None):
        """Mixed-structure batch (kgq_submit_mixed) -> global top-k: the local [sum B_i, k]
        lists are all-gathered and merged exactly like a single-structure submit."""
        td, ti = self.engine.submit_mixed(groups, k, stream=stream)
        self._launches = self.engine.last_launch_count()
        if self.world == 1:
            return td, ti
        self._launches += 1  # the merge kernel (NCCL's own kernels are not counted)
        if self.merge_mode == "p2p":
            return self.engine.merge_peers(td.shape[0], k, stream=stream)
        gd, gi = all_gather_topk(td, ti, self.group)
        return self.engine.merge_topk(gd, gi, k, stream=stream)

    def last_launch_count(self):
        return self._launches

    def rank_answers(self, structure, anchors, rels, ans_off, ans_id, stream=None):
        """N1 filtered ranks (1-based) of every answer across all shards: answer distances
        from the owning shard (min-all-reduce of +inf elsewhere), then per-shard counts of
        better non-answers, sum-all-reduced."""
        if self.world == 1:
            _, cnt = self.engine.rank_answers(structure, anchors, rels, ans_off, ans_id, RANK_LOCAL,
                                              stream=stream)
            return cnt + 1
        ad, _ = self.engine.rank_answers(structure, anchors, rels, ans_off, ans_id, RANK_DIST,
                                         stream=stream)
        dist.all_reduce(ad, op=dist.ReduceOp.MIN, group=self.group)
        _, cnt = self.engine.rank_answers(structure, anchors, rels, ans_off, ans_id, RANK_COUNT,
                                          ans_dist=ad, stream=stream)
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=self.group)
        return cnt + 1


def answers_csr(answer_lists):
    """[array of global ids per query] -> (ans_off int32 [B+1], ans_id int32 [n]) numpy."""
    import numpy as np
    off = np.zeros(len(answer_lists) + 1, np.int32)
    off[1:] = np.cumsum([len(a) for a in answer_lists])
    ids = np.concatenate([np.asarray(a, np.int32) for a in answer_lists]) if answer_lists else np.zeros(0, np.int32)
    return off, ids.astype(np.int32)


def mrr_hits(ranks_per_query):
    """Mean over queries of the per-query mean of 1/rank and Hits@1/3/10 over its hard answers."""
    import numpy as np
    m = np.array([[np.mean(1.0 / r), np.mean(r <= 1), np.mean(r <= 3), np.mean(r <= 10)]
                  for r in (np.asarray(x, np.float64) for x in ranks_per_query) if len(r)])
    return dict(zip(("mrr", "hits1", "hits3", "hits10"), m.mean(0).tolist())) if len(m) else {}
