"""N2 timing on one GPU (not part of the library): W virtual entity shards of the FB15k-237-shape
BetaE model at batch 1024, k = 10.  Device time (CUDA events) of
  - one rank's submit without / with the fused peer push (the top-k writes its rows into all W
    peer buffers and releases the row flags),
  - kgq_merge_peers (wait + W-way merge) vs kgq_merge_topk (the merge kernel the NCCL path runs
    after its all-gather; the all-gather itself needs W GPUs and is not timed here).
On one GPU the peer buffers are local HBM, so the push cost is a lower bound of the NVLink one."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2503_02172_b200 import Engine  # noqa: E402

N, R, D, H, B, K = 14505, 237, 400, 1600, 1024, 10


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    t = synth.make_tables("betae", N, R, D, hidden=H, seed=1)
    a, r = synth.make_queries("1p", B, N, R, seed=2)
    da = torch.from_numpy(a.astype(np.int32)).cuda()
    dr = torch.from_numpy(r.astype(np.int32)).cuda()
    out = {}
    for W in (2, 8):
        engs = [Engine("betae", N, R, D, hidden=H, max_batch=B, max_k=K, world_size=W, rank=q) for q in range(W)]
        for e in engs:
            e.load_tables(t)
        e0 = engs[0]
        td = torch.empty((B, K), dtype=torch.float32, device="cuda")
        ti = torch.empty((B, K), dtype=torch.int32, device="cuda")
        plain = timed(lambda: e0.submit("1p", da, dr, K, out=(td, ti)))
        bufs = [torch.empty(e0.peer_bytes(W), dtype=torch.uint8, device="cuda") for _ in range(W)]
        for q, e in enumerate(engs):
            e.set_peers(q, W, [b.data_ptr() for b in bufs])
        outs = [(torch.empty_like(td), torch.empty_like(ti)) for _ in range(W)]
        md = (torch.empty_like(td), torch.empty_like(ti))

        def all_push():
            for q, e in enumerate(engs):
                e.submit("1p", da, dr, K, out=outs[q])

        pushed = timed(lambda: e0.submit("1p", da, dr, K, out=outs[0]))
        for q, e in enumerate(engs):  # rank 0 ran ahead: reset every epoch and buffer
            e.set_peers(q, W, [b.data_ptr() for b in bufs])
        # rounds of: every rank pushes, then every rank merges (a merge advances its epoch);
        # rank 0's merge timed alone
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(23)]
        for a0, a1 in ev:
            all_push()
            a0.record()
            e0.merge_peers(B, K, out=md)
            a1.record()
            for e in engs[1:]:
                e.merge_peers(B, K)
        torch.cuda.synchronize()
        merge_p2p = float(np.mean([a0.elapsed_time(a1) for a0, a1 in ev[3:]])) * 1e3
        gd = torch.stack([o[0] for o in outs])
        gi = torch.stack([o[1] for o in outs])
        merge_nccl_kernel = timed(lambda: e0.merge_topk(gd, gi, K))
        for e in engs:
            e.check_errors()
            e.close()
        out[W] = {"submit_us": plain, "submit_with_push_us": pushed, "merge_peers_us": merge_p2p,
                  "merge_topk_kernel_us": merge_nccl_kernel}
        print(f"W={W}: submit {plain:.1f} us, with fused push {pushed:.1f} us; merge_peers {merge_p2p:.1f} us "
              f"(all pushes done), merge_topk kernel {merge_nccl_kernel:.1f} us", flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
