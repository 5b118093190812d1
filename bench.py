#!/usr/bin/env python
"""Benchmark of the CLQA inference hot path (BASELINE.json metric).

Workload (N=1): BASELINE.json configs[1] -- BetaE on the synthetic FB15k-237 shape
(14,505 entities, 237 relations, d 400, MLP 1600x2), batch 1024, all 14 query types.
One step = one batch of every query type through the whole path (operator chain ->
entity scoring -> top-k 10), i.e. 14 x 1024 queries, submitted as ONE kgq_submit_mixed
(default; --mode per-type: 14 kgq_submit calls over --streams streams).  value = queries/s
over all ranks; "per_type" gives each type's own queries/s (the metric's per-type view).

N > 1 (torchrun): --split queries (default): a W x 14 x 1024 replicated batch, each rank runs its
own 14 x 1024 queries and the library's NCCL all-gather returns the whole batch's top-k (weak
scaling); --split entities: the entity table is sharded, every rank scores the replicated batch
on its shard, local top-k + all-gather + merge inside the library (strong scaling).

--impl reference: the float64 CPU oracle (the reference arm of this tier), on rank 0 only.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "queries/sec per query type (BetaE, FB15k-237 shape) at 1/2/4/8 B200; HBM GB/s"
N_ENT, N_REL, DIM, HID, BATCH, K = 14505, 237, 400, 1600, 1024, 10
SEED = 2503_02172 + 1
STRUCTS = synth.STRUCTURES
CONFIG = {
    "workload": "BetaE FB15k-237 shape, all 14 query types (BASELINE.json configs[1])",
    "n_entity": N_ENT, "n_relation": N_REL, "dim": DIM, "hidden": HID, "hidden_layers": 2,
    "batch": BATCH, "k": K, "structures": list(STRUCTS), "inputs": "kgr-init (random-init), seed 2503021173",
}


def operand_format(mmas):
    return {3: "fp16x2", 6: "bf16x3"}.get(mmas, f"{mmas}-MMA")


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            out, _ = self.p.communicate(timeout=5)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "samples": len(sm), "reasons": sorted(reasons)}


def timed_oracle_sample(n_queries, start_type=0):
    """The float64 oracle on `n_queries` BetaE queries (types cycling) -> (seconds, queries)."""
    import oracle
    t = synth.make_tables("betae", N_ENT, N_REL, DIM, hidden=HID, seed=SEED)
    m = oracle.Model("betae", t, dim=DIM)
    t0 = time.perf_counter()
    for i in range(n_queries):
        s = STRUCTS[(start_type + i) % len(STRUCTS)]
        a, r = synth.make_queries(s, 1, N_ENT, N_REL, seed=synth.query_seed(SEED, s))
        oracle.answer(m, s, a, r, K)
    return time.perf_counter() - t0, n_queries


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return 1


def run_reference(args, rank, world):
    if rank != 0:
        return
    # warmup steps, then K timed steps; each step = one oracle query (types cycling)
    timed_oracle_sample(args.warmup, 0)
    sec, n = timed_oracle_sample(args.steps, args.warmup)
    v = n / sec
    cores = blas_threads()
    line = {"metric": METRIC, "value": v, "unit": "queries/s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sec / max(1, args.steps), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": CONFIG,
            "cpu_baseline": {"value": v, "unit": "queries/s", "cores": cores, "kind": "oracle",
                             "sample": f"{n} BetaE queries (1 per step, types cycling), full "
                                       f"14,505-entity literal-KL scoring + sort, float64 numpy"},
            "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def c5a_measure(steps, warmup, peaks, models=("gqe", "betae")):
    """BASELINE.json configs[4], latency regime: 2M entities, d 400, GQE and
    BetaE, B in {1, 8}, 1p and 2u, one GPU.  The dominant kernel is the streaming entity scorer
    (k_score_stream): its algorithmic bytes per launch are the shard's scoring table read once
    (GQE: 4 N d bytes; BetaE: the C, U, V planes, 12 N d bytes), its time the library's stage
    events around the scorer launch (one kernel, ~0.5-1.7 ms: the event nodes cost < 1%)."""
    import torch
    from paper_2503_02172_b200 import Engine
    N, R, d = 2_000_000, 200, 400
    res = {}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for model in models:
        t = synth.make_tables(model, N, R, d, hidden=HID, seed=77)
        eng = Engine(model, N, R, d, hidden=HID, max_batch=8, max_k=K)
        eng.load_tables(t)
        del t
        # the table the scorer streams: GQE [d][N] fp32; BetaE the centred (u, v) planes [d][2][N]
        # (KGQ_BETAE_STREAM=cuv: the round-1 C, U, V planes [d][3][N])
        planes = 1 if model == "gqe" else (3 if os.environ.get("KGQ_BETAE_STREAM", "").startswith("c") else 2)
        table_bytes = planes * d * 4 * (eng.shard[1] - eng.shard[0])
        for s in ("1p", "2u"):
            for B in (1, 8):
                a, r = synth.make_queries(s, B, N, R, seed=5)
                da, dr = torch.from_numpy(a).cuda(), torch.from_numpy(r).cuda()
                for _ in range(warmup):
                    eng.submit(s, da, dr, K)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

                def c5a_steps():
                    tt = 0.0
                    for _ in range(steps):
                        flush.zero_()
                        e0.record()
                        eng.submit(s, da, dr, K)
                        e1.record()
                        torch.cuda.synchronize()
                        tt += e0.elapsed_time(e1)
                    return tt
                tot = c5a_steps()  # whole submits, no stage events
                eng.profile(True)  # second pass: the scorer's own time
                eng.submit(s, da, dr, K)
                eng.submit(s, da, dr, K)
                torch.cuda.synchronize()
                eng.profile_read()
                c5a_steps()
                prof = eng.profile_read()
                eng.profile(False)
                sc_ms = prof["score"][0] / max(1, prof["score"][1])
                gbs = table_bytes / (sc_ms / 1e3) / 1e9
                # FP32 lane operations per (entity, dim) of the scorer's inner loop: GQE |e - q| and
                # the sum (2 per query row), BetaE a u + b v (2 FMAs per query row); rows = B x branches
                rows = B * (2 if s == "2u" else 1)
                ops = 2 * rows * N * d
                alu_peak = 148 * 128 * peaks.get("sm_max_mhz", 1965.0) * 1e6
                alu = ops / (sc_ms / 1e3)
                res[f"{model}_{s}_B{B}"] = {
                    "ms_per_batch": tot / steps, "queries_per_s": B * steps / (tot / 1e3),
                    "scorer_ms": sc_ms, "scorer_table_gbs": gbs, "hbm_frac": gbs / peaks["hbm_gbs"],
                    "alu_tops": alu / 1e12, "alu_frac": alu / alu_peak,
                    # the binding roof: the one the kernel would hit first at 100%
                    "bound": "hbm" if table_bytes / (peaks["hbm_gbs"] * 1e9) >= ops / alu_peak else "alu",
                }
        eng.close()
    return res


def run_c5a(args):
    peaks, src = load_peaks()
    res = c5a_measure(args.steps, args.warmup, peaks, tuple(args.models.split(",")))
    print(json.dumps({"metric": "C5a latency regime: 2M-entity scoring HBM GB/s (1 GPU)",
                      "hbm_peak_gbs": peaks["hbm_gbs"], "peak_source": src, "results": res}), flush=True)


SUITE = {
    # name: (model, N, R, d, hidden, batch, structures, note) -- BASELINE.json configs
    "c1_gqe_toy": ("gqe", 200, 10, 32, 64, 16, ("1p", "2p", "2i"), "configs[0]: GQE toy KG, latency regime"),
    "c3_q2b_nell995": ("q2b", 63361, 200, 400, 1600, 1024, ("1p", "2p", "3p", "2i", "3i", "pi", "ip", "2u", "up"),
                       "configs[2]: Query2Box EPFO types on the NELL995 shape"),
    "c4_betae_fb15k_neg": ("betae", 14951, 1345, 400, 1600, 4096, ("2in", "3in", "inp", "pin", "pni"),
                           "configs[3]: BetaE negation types on the FB15k shape, batch 4096"),
    "c5b_gqe_2m": ("gqe", 2_000_000, 200, 400, 1600, 1024, ("1p", "2u"), "configs[4], throughput regime B=1024"),
    "c5b_betae_2m": ("betae", 2_000_000, 200, 400, 1600, 1024, ("1p", "2u"), "configs[4], throughput regime B=1024"),
}


def run_suite(args):
    """One JSON line per BASELINE.json config other than the headline one: device
    q/s with L2 flushed between steps, stage split, and the dominant kernel against its roofline
    (SIMT scorers: FP32 lane-instructions vs 148 SMs x 128 lanes x SM clock; tensor path: useful
    fp32 FLOPs vs the tensor peak = measured bf16 (= fp16) / MMAs per fp32 FMA of the build)."""
    import torch
    from paper_2503_02172_b200 import Engine
    peaks, src = load_peaks()
    alu_peak = 148 * 128 * peaks.get("sm_max_mhz", 1965.0) * 1e6  # lane-instr/s
    from paper_2503_02172_b200.kgq import tensor_mmas_per_fma
    mmas = tensor_mmas_per_fma()
    tc_peak = peaks["bf16_tflops"] / mmas
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    names = args.suite.split(",") if args.suite else list(SUITE)
    for name in names:
        model, N, R, d, H, B, structs, note = SUITE[name]
        t = synth.make_tables(model, N, R, d, hidden=H, seed=SEED + 10)
        eng = Engine(model, N, R, d, hidden=H, max_batch=B, max_k=K)
        eng.load_tables(t)
        del t
        qs = {}
        for s in structs:
            a, r = synth.make_queries(s, B, N, R, seed=synth.query_seed(SEED + 10, s))
            qs[s] = (torch.from_numpy(a).cuda(), torch.from_numpy(r).cuda())
        for _ in range(args.warmup):
            for s in structs:
                eng.submit(s, *qs[s], K)
        torch.cuda.synchronize()
        eng.check_errors()
        ev = {s: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for s in structs}

        def suite_steps():
            per = {s: 0.0 for s in structs}
            for _ in range(args.steps):
                flush.zero_()
                torch.cuda.synchronize()
                for s in structs:
                    ev[s][0].record()
                    eng.submit(s, *qs[s], K)
                    ev[s][1].record()
                torch.cuda.synchronize()
                for s in structs:
                    per[s] += ev[s][0].elapsed_time(ev[s][1])
            return per
        per = suite_steps()  # headline: no stage events
        eng.profile(True)    # second pass: stage split + scorer / GEMM times
        for s in structs:    # capture the profiled graphs before the pass
            eng.submit(s, *qs[s], K)
            eng.submit(s, *qs[s], K)
        torch.cuda.synchronize()
        eng.profile_read()
        suite_steps()
        prof = eng.profile_read()
        eng.profile(False)
        eng.close()
        mixed = None
        if model == "betae" and len(structs) > 1:
            # the same queries as ONE kgq_submit_mixed (level-synchronous batching across the
            # types, the headline's step form), L2 flushed before each step, device time
            meng = Engine(model, N, R, d, hidden=H, max_batch=B * len(structs), max_k=K)
            meng.load_tables(synth.make_tables(model, N, R, d, hidden=H, seed=SEED + 10))
            pa = torch.cat([qs[s][0].reshape(-1) for s in structs]).int().contiguous()
            pr = torch.cat([qs[s][1].reshape(-1) for s in structs]).int().contiguous()
            mo = (torch.empty((B * len(structs), K), device="cuda"),
                  torch.empty((B * len(structs), K), dtype=torch.int32, device="cuda"))
            bl = [B] * len(structs)
            for _ in range(max(args.warmup, 2)):
                meng.submit_mixed_packed(list(structs), bl, pa, pr, K, mo)
            torch.cuda.synchronize()
            meng.check_errors()
            mt = 0.0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(args.steps):
                flush.zero_()
                torch.cuda.synchronize()
                e0.record()
                meng.submit_mixed_packed(list(structs), bl, pa, pr, K, mo)
                e1.record()
                torch.cuda.synchronize()
                mt += e0.elapsed_time(e1)
            meng.check_errors()
            meng.close()
            mixed = {"form": f"one kgq_submit_mixed of the {len(structs)} x {B} queries per step",
                     "queries_per_s": args.steps * len(structs) * B / (mt / 1e3), "ms_per_step": mt / args.steps}
        tot = sum(per.values())
        q = args.steps * len(structs) * B
        st = {k: v[0] / args.steps for k, v in prof.items()}
        sc_ms, _, sc_w = prof["score"]
        d_ms, _, d_w = prof["dense"]
        if model == "betae" and B > 16:
            ach = (sc_w + d_w) / ((sc_ms + d_ms) / 1e3) / 1e12
            roof = {"kernel": f"k_gemm (tcgen05, {operand_format(mmas)} operands: dense layers + BetaE scorer)",
                    "bound": "tensor",
                    "achieved": ach, "peak": tc_peak, "unit": "TFLOP/s", "frac": ach / tc_peak}
        else:
            ach = sc_w / (sc_ms / 1e3) if sc_ms > 0 else 0.0
            roof = {"kernel": f"k_score<{model}> (SIMT L1 / box distance)", "bound": "alu",
                    "achieved": ach / 1e12, "peak": alu_peak / 1e12, "unit": "T lane-instr/s",
                    "frac": ach / alu_peak}
        print(json.dumps({"workload": name, "note": note, "model": model, "n_entity": N, "n_relation": R,
                          "dim": d, "batch": B, "k": K, "structures": list(structs),
                          "queries_per_s": q / (tot / 1e3), "ms_per_batch": tot / args.steps / len(structs),
                          "per_type_qps": {s: B * args.steps / (per[s] / 1e3) for s in structs},
                          "stage_ms_per_step": st, "roofline": roof, "peak_source": src,
                          "mixed_submit": mixed, "l2": "flushed between steps"}), flush=True)


def span_union_ms(spans):
    """Length of the union of [start, end) intervals (ns) -> ms."""
    if len(spans) == 0:
        return 0.0
    iv = sorted((int(a), int(b)) for a, b in spans)
    tot, cs, ce = 0, iv[0][0], iv[0][1]
    for a, b in iv[1:]:
        if a > ce:
            tot += ce - cs
            cs, ce = a, b
        else:
            ce = max(ce, b)
    return (tot + ce - cs) * 1e-6


def replicated_groups(world, qsplit):
    """The step's query groups: (structure, rows, anchors, rels) in submit order.  N = 1 or the
    entity split: one group of BATCH queries per structure.  Query split: W x 14 groups, rank w's
    14 groups (its own seeds) contiguous, so the library's row range [w Q, (w+1) Q) of the
    replicated batch is exactly rank w's 14 x 1024 queries (the same mix of types on every rank)."""
    out = []
    for w in range(world if qsplit else 1):
        for s in STRUCTS:
            a, r = synth.make_queries(s, BATCH, N_ENT, N_REL, seed=synth.query_seed(SEED, s) + 7919 * w)
            out.append((s, BATCH, a.astype(np.int32), r.astype(np.int32)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kgq", choices=["kgq", "reference"])
    ap.add_argument("--mode", default="mixed", choices=["mixed", "per-type"],
                    help="headline step: ONE kgq_submit_mixed of the 14 x 1024 queries (each projection hop of "
                         "every type is one MLP), or the 14 per-type kgq_submit calls dealt over --streams streams")
    ap.add_argument("--streams", type=int, default=3,
                    help="per-type mode: concurrent streams per GPU (one library context each)")
    ap.add_argument("--split", default="queries", choices=["queries", "entities"],
                    help="N>1: rank r runs its 14 x 1024 queries of a W x 14 x 1024 replicated batch (weak scaling, "
                         "the library's query-split communicator), or the entity table is sharded over the ranks "
                         "with a replicated 14 x 1024-query batch (strong scaling, local top-k + all-gather + merge)")
    ap.add_argument("--merge", default="nccl", choices=["nccl", "p2p", "torch"],
                    help="entity split: the library's NCCL all-gather + merge kernel (default), the all-gather "
                         "fused into the top-k over symmetric peer memory (N2), or torch.distributed + merge")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-queries", type=int, default=14)
    ap.add_argument("--no-per-type", action="store_true",
                    help="skip the secondary per-type measurements (14 submits over streams; each type alone)")
    ap.add_argument("--no-mixed", action="store_true", help=argparse.SUPPRESS)  # round-1 flag, = --no-per-type
    ap.add_argument("--no-c5a", action="store_true", help="skip the 2M-entity HBM (C5a) measurement")
    ap.add_argument("--workload", default="fb15k237", choices=["fb15k237", "c5a", "suite"])
    ap.add_argument("--suite", default="", help="comma list of SUITE configs (default: all)")
    ap.add_argument("--models", default="gqe,betae", help="--workload c5a: models to measure")
    args = ap.parse_args()
    if args.workload == "c5a":
        return run_c5a(args)
    if args.workload == "suite":
        return run_suite(args)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2503_02172_b200 import Engine
    from paper_2503_02172_b200.sharded import ShardedEngine

    # KGQ_BENCH_ONE_GPU=1 (testing the N > 1 code path on a one-GPU box only): every rank on
    # cuda:0 with the gloo backend and merge="torch" -- the numbers of such a run mean nothing
    one_gpu = os.environ.get("KGQ_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    mixed_mode = args.mode == "mixed"
    S = 1 if mixed_mode else max(1, args.streams)
    # the query split runs through the library's NCCL communicator, which needs one GPU per rank:
    # the one-GPU path check uses the entity split with the torch.distributed merge instead
    qsplit = world > 1 and args.split == "queries" and not one_gpu
    merge = "nccl" if qsplit else (args.merge if not one_gpu else "torch")
    t = synth.make_tables("betae", N_ENT, N_REL, DIM, hidden=HID, seed=SEED)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    main_stream = torch.cuda.current_stream()
    per_rank_queries = len(STRUCTS) * BATCH  # per step (query split: each rank's own rows)
    job_queries = per_rank_queries * (world if qsplit else 1)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(vals):
        if world == 1:
            return vals
        tt = torch.tensor(vals, dtype=torch.float64, device="cuda" if not one_gpu else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return [float(x) for x in tt.tolist()]

    # ---------------- the step's queries ----------------
    groups = replicated_groups(world, qsplit)
    Qg = sum(g[1] for g in groups)                      # replicated batch per step
    g_structs, g_batches = [g[0] for g in groups], [g[1] for g in groups]
    a_host = np.concatenate([g[2].reshape(-1) for g in groups])
    r_host = np.concatenate([g[3].reshape(-1) for g in groups])
    a_dev, r_dev = torch.from_numpy(a_host).cuda(), torch.from_numpy(r_host).cuda()

    # ---------------- headline engines ----------------
    launches = [0]
    if mixed_mode:
        se = ShardedEngine("betae", N_ENT, N_REL, DIM, split="queries" if qsplit else "entities", hidden=HID,
                           max_batch=Qg, max_k=K, device=local, merge=merge)
        se.load_tables(t)
        se.p2p_check = False  # N2 errors are checked once after the timed steps
        engines = [se]
        mout = (torch.empty((Qg, K), device="cuda"), torch.empty((Qg, K), dtype=torch.int32, device="cuda"))
        streams = [main_stream]

        def submit_all(nlanes=1, count=True):
            se.submit_mixed_packed(g_structs, g_batches, a_dev, r_dev, K, mout, stream=main_stream)
            if count:
                launches[0] += se.last_launch_count()
    else:
        engines = []
        for _ in range(S):
            e = ShardedEngine("betae", N_ENT, N_REL, DIM, split="queries" if qsplit else "entities", hidden=HID,
                              max_batch=BATCH * (world if qsplit else 1), max_k=K, device=local, merge=merge)
            e.load_tables(t)
            e.p2p_check = False
            engines.append(e)
        streams = [torch.cuda.Stream() for _ in range(S)]
        # per type: the W x 1024 replicated rows in rank order (query split), else the 1024
        per_type_in = {}
        for s in STRUCTS:
            sel = [g for g in groups if g[0] == s]
            per_type_in[s] = (torch.from_numpy(np.concatenate([g[2] for g in sel])).cuda(),
                              torch.from_numpy(np.concatenate([g[3] for g in sel])).cuda())
        lane = {s: i % S for i, s in enumerate(STRUCTS)}

        def submit_all(nlanes=S, count=True):
            for s in STRUCTS:
                j = lane[s] % nlanes
                engines[j].submit(s, *per_type_in[s], K, stream=streams[j])
                if count:
                    launches[0] += engines[j].last_launch_count()
    for se_ in engines:
        se_.engine.ktime(True)  # in-kernel GEMM launch spans (roofline from this very pass)

    def step(nlanes=S, count=True):
        """One step (all 14 x 1024 queries of this rank) between two events on the main stream
        (per-type mode: forked over `nlanes` streams and joined before the end event)."""
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(main_stream)
        for st in streams[:nlanes]:
            if st is not main_stream:
                st.wait_event(e0)
        submit_all(nlanes, count)
        for st in streams[:nlanes]:
            if st is not main_stream:
                ev = torch.cuda.Event()
                ev.record(st)
                main_stream.wait_event(ev)
        e1.record(main_stream)
        return e0, e1

    def timed(nsteps, nlanes):
        """nsteps steps, L2 flushed (untimed) before each; per-step device ms."""
        ms = []
        for _ in range(nsteps):
            flush.zero_()
            e0, e1 = step(nlanes)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return ms

    for _ in range(max(3, args.warmup)):
        step(S, False)
        if S > 1:
            step(1, False)  # the sequential pass's graphs (lane 0) are captured here too
    barrier()
    for se_ in engines:
        se_.engine.check_errors()
        se_.engine.ktime_read()
        se_.engine.ktime_log()
    launches[0] = 0
    with ClockSampler(local) as clk:
        barrier()
        step_ms = timed(args.steps, S)
        barrier()
    n_launch = launches[0]
    logs = [se_.engine.ktime_log() for se_ in engines]
    for se_ in engines:
        se_.engine.ktime_read()
    spans = np.concatenate([lg for lg in logs if len(lg)]) if any(len(lg) for lg in logs) else np.zeros((0, 3), np.uint64)
    gemm_busy_ms = span_union_ms(spans[:, :2]) / args.steps
    dense_busy_ms = span_union_ms(spans[spans[:, 2] == 0][:, :2]) / args.steps
    score_busy_ms = span_union_ms(spans[spans[:, 2] == 1][:, :2]) / args.steps
    gemm_launches = len(spans) / args.steps
    total_ms = sum(step_ms)
    seq_ms = seq_dense_ms = seq_score_ms = None
    if S > 1:  # per-type mode: the same steps on ONE stream (each GEMM alone on the GPU)
        barrier()
        seq_ms = sum(timed(args.steps, 1))
        lg = engines[0].engine.ktime_log()
        seq_dense_ms = span_union_ms(lg[lg[:, 2] == 0][:, :2]) / args.steps
        seq_score_ms = span_union_ms(lg[lg[:, 2] == 1][:, :2]) / args.steps
        for se_ in engines:
            se_.engine.ktime_log()
            se_.engine.ktime_read()
    total_ms, seq_ms = max_over_ranks([total_ms, seq_ms or 0.0])
    seq_ms = seq_ms or None
    value = job_queries * args.steps / (total_ms / 1e3)
    for se_ in engines:
        se_.engine.check_errors()

    # ---- algorithmic GEMM FLOPs per step (the library's own work counters, one profiled
    # step outside the timed region; this rank's rows) ----
    for se_ in engines:
        se_.engine.ktime(False)
        se_.engine.profile(True)
        se_.engine.profile_read()
    step(1, False)
    torch.cuda.synchronize()
    d_fl = s_fl = 0.0
    for se_ in engines:
        prof = se_.engine.profile_read()
        se_.engine.profile(False)
        d_fl += prof["dense"][2]
        s_fl += prof["score"][2]

    # ---- secondary (1 GPU): the other step form, and every type alone ----
    other = per_type = None
    if world == 1 and not (args.no_per_type or args.no_mixed):
        try:
            other, per_type = secondary_passes(args, t, groups, mixed_mode, flush)
        except Exception as ex:
            print(f"bench: secondary passes failed: {type(ex).__name__}: {ex}", file=sys.stderr, flush=True)

    # ---- end to end through the public API with host buffers (pinned) ----
    e2e_v = None
    h2d = (a_host.size + r_host.size) * 4
    d2h = Qg * K * 8
    try:
        if mixed_mode and engines[0].merge_mode in ("local", "nccl"):
            pa, pr = torch.from_numpy(a_host).pin_memory(), torch.from_numpy(r_host).pin_memory()
            hd, hi = torch.empty((Qg, K)).pin_memory(), torch.empty((Qg, K), dtype=torch.int32).pin_memory()

            def e2e_step():
                engines[0].submit_mixed_host(g_structs, g_batches, pa.numpy(), pr.numpy(), K,
                                             (hd.numpy(), hi.numpy()), stream=main_stream)
                main_stream.synchronize()
            e2e_how = ("per step: one kgq_submit_mixed_host_async (pinned H2D of the packed anchors / relations, "
                       "the whole path, D2H of the top-k into pinned host outputs), stream synchronised")
        else:
            pin = {}
            for s in STRUCTS:
                sel = [g for g in groups if g[0] == s]
                pin[s] = (torch.from_numpy(np.concatenate([g[2] for g in sel])).pin_memory(),
                          torch.from_numpy(np.concatenate([g[3] for g in sel])).pin_memory())
            nrow = BATCH * (world if qsplit else 1)
            hout = {s: (torch.empty((nrow, K)).pin_memory(), torch.empty((nrow, K), dtype=torch.int32).pin_memory())
                    for s in STRUCTS}
            lane_e = {s: i % len(engines) for i, s in enumerate(STRUCTS)}
            e2e_streams = streams if not mixed_mode else [main_stream]

            def e2e_step():
                for s in STRUCTS:
                    j = lane_e[s]
                    engines[j].engine.submit_host(s, pin[s][0].numpy(), pin[s][1].numpy(), K,
                                                  out=(hout[s][0].numpy(), hout[s][1].numpy()),
                                                  stream=e2e_streams[j % len(e2e_streams)], sync=False)
                for st in e2e_streams:
                    st.synchronize()
            e2e_how = (f"per step: kgq_submit_host_async per type on {len(e2e_streams)} stream(s) (pinned H2D, path, "
                       f"D2H of the top-k into pinned host outputs), every stream synchronised")
        e2e_step()
        e2e_step()
        e2e_s = 0.0
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            t0 = time.perf_counter()
            e2e_step()
            e2e_s += time.perf_counter() - t0
        e2e_s = max_over_ranks([e2e_s])[0]
        e2e_v = job_queries * args.steps / e2e_s
    except Exception as ex:  # a failure here must not cost the headline line: e2e is then null
        e2e_how = f"failed: {type(ex).__name__}: {ex}"
        print(f"bench: e2e failed: {type(ex).__name__}: {ex}", file=sys.stderr, flush=True)
    for se_ in engines:
        se_.engine.check_errors()

    # ---- C5a: the north-star HBM target (2M-entity scoring sweep, B in {1, 8}) ----
    peaks, peak_src = load_peaks()
    c5a = None
    if world == 1 and not args.no_c5a:
        try:
            c5a = c5a_measure(max(3, args.steps // 2), 2, peaks)
        except Exception as ex:
            print(f"bench: C5a failed: {type(ex).__name__}: {ex}", file=sys.stderr, flush=True)

    # ---- roofline of the dominant kernel: the tcgen05 GEMM (k_gemm), which runs every
    # dense layer of the chain and the BetaE scorer contraction.  Algorithmic work = useful fp32
    # FLOPs (2MNK, the library's counters); time = the union of the GEMM launches' in-kernel spans
    # (%globaltimer, first CTA start after the PDL wait -> last CTA end) over the timed steps of
    # THIS pass; peak = measured bf16 (fp16 MMAs run at the same rate) / the build's MMAs per
    # useful fp32 multiply-add (fp16x2: a_h w_h' + a_h w_l' + a_l' w_h = 3; bf16x3: 6), the BURST
    # figure (the driver's sustained one is a 4-s cuBLAS loop under the power cap), sustained
    # quoted beside.
    from paper_2503_02172_b200.kgq import tensor_mmas_per_fma
    mmas = tensor_mmas_per_fma()  # 3: fp16x2 operands (default build), 6: bf16x3 (libkgq_bf16x3.so)
    peak_sus = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) / mmas
    peak_burst = peaks["bf16_tflops"] / mmas
    rate = lambda fl, ms: fl / (ms / 1e3) / 1e12 if ms and ms > 0 else 0.0
    achieved = rate(d_fl + s_fl, gemm_busy_ms)
    traffic = None
    tf = os.path.join(ROOT, "profiles", "tc_gemm_traffic.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get("dram_bytes_per_launch")
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    ms_step = total_ms / args.steps
    # parts: each part's GEMMs alone on the GPU -- the headline pass itself in mixed mode (one
    # stream: the launches run one after another), the sequential pass in per-type mode
    p_dense, p_score = (dense_busy_ms, score_busy_ms) if S == 1 else (seq_dense_ms, seq_score_ms)
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak" if qsplit or world == 1 else "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": dict(CONFIG, l2="flushed between timed steps (256 MiB write, untimed)",
                       step="mixed" if mixed_mode else f"per-type x {S} streams",
                       parallelism=("1 GPU" if world == 1 else
                                    f"query split x{world} (W x 14 x 1024 replicated queries, each rank its 14 x "
                                    f"1024; library NCCL all-gather)" if qsplit else
                                    f"entity shards x{world} ({engines[0].merge_mode})"),
                       queries_per_step_per_rank=per_rank_queries,
                       gemm_operands=("fp16x2 split: fp32 operands as fp16 hi + 2^11-scaled fp16 lo, 3 fp16 MMAs "
                                      "per fp32 multiply-add, fp32 accumulation (DESIGN.md §7)" if mmas == 3 else
                                      "bf16x3 split: exact three bf16 planes, 6 MMAs per fp32 multiply-add")),
        "how": ("per step: ONE kgq_submit_mixed of the 14 x 1024 queries (BetaE level-synchronous: each projection "
                "hop of all types' branches is one MLP, all intersections one attention GEMM pair, later branch hops "
                "batched with the post-intersection hops, one scorer, one top-k); device time between events on the launching stream, max over ranks" if mixed_mode else
                f"per step: the 14 per-type kgq_submit calls dealt round-robin over {S} CUDA streams, one library "
                f"context per stream; device time from an event before the fork to an event after the join, max "
                f"over ranks"),
        "per_type": per_type,
        "other_step_form": other,
        "sequential": None if seq_ms is None else {
            "value": job_queries * args.steps / (seq_ms / 1e3), "ms_per_step": seq_ms / args.steps,
            "how": "the same steps with the 14 submits on one stream (no overlap between types)"},
        "gemm": {"busy_ms_per_step": gemm_busy_ms, "dense_busy_ms_per_step": dense_busy_ms,
                 "score_busy_ms_per_step": score_busy_ms, "launches_per_step": gemm_launches,
                 "share_of_step": gemm_busy_ms / ms_step,
                 "how": "in-kernel %globaltimer spans of every k_gemm launch of the timed steps (kgq_ktime_log), "
                        "union over the streams"},
        "roofline": {"kernel": f"k_gemm (tcgen05, {operand_format(mmas)} operands: chain dense layers + BetaE scorer)",
                     "bound": "tensor", "achieved": achieved, "peak": peak_burst, "unit": "TFLOP/s",
                     "frac": achieved / peak_burst, "traffic": traffic,
                     "peak_source": f"{peak_src} bf16 burst {peak_burst * mmas:.1f} TFLOP/s (fp16 MMAs run at the bf16 "
                                    f"rate) / {mmas} ({operand_format(mmas)}: {mmas} MMAs per useful fp32 multiply-add)",
                     "frac_vs_sustained": achieved / peak_sus,
                     "work": f"useful fp32 FLOPs 2MNK per GEMM launch: {(d_fl + s_fl) / 1e9:.1f} GFLOP per step "
                             f"per rank (dense {d_fl / 1e9:.1f}, score {s_fl / 1e9:.1f})",
                     "whole_step_rate": rate(d_fl + s_fl, ms_step),
                     "parts": None if not p_dense else {
                         "how": "each part's GEMMs alone on the GPU (in-kernel spans)",
                         "dense": {"ms_per_step": p_dense, "tflops": rate(d_fl, p_dense),
                                   "frac": rate(d_fl, p_dense) / peak_burst},
                         "score": {"ms_per_step": p_score, "tflops": rate(s_fl, p_score),
                                   "frac": rate(s_fl, p_score) / peak_burst}}},
        "gpu_launches": n_launch,
        "e2e": {"value": e2e_v, "unit": "queries/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "how": e2e_how + "; wall clock, L2 flushed before each step (untimed), max over ranks"},
        "hbm": None if c5a is None else {
            "workload": "BASELINE.json configs[4] latency regime: 2M entities, d 400, 1 GPU, GQE / BetaE, "
                        "1p / 2u, B in {1, 8}",
            "kernel": "k_score_stream / k_score_uv_stream (streaming entity scorers)", "bound": "hbm",
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "peak_source": f"{peak_src} copy bandwidth",
            "work": "the shard's scoring table read once per batch: GQE 4 N d bytes, BetaE 8 N d (the centred "
                    "fp32 u, v planes)",
            "alu_peak": "148 SMs x 128 FP32 lanes x max SM clock (FFMA2 / FADD2 counted per lane operation)",
            "results": {k: {"gbs": round(v["scorer_table_gbs"], 1), "frac": round(v["hbm_frac"], 4),
                            "alu_frac": round(v["alu_frac"], 4), "bound": v["bound"],
                            "frac_of_bound": round(v["hbm_frac"] if v["bound"] == "hbm" else v["alu_frac"], 4),
                            "queries_per_s": round(v["queries_per_s"], 1)} for k, v in c5a.items()}},
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        sec, n = timed_oracle_sample(args.cpu_queries, 0)
        line["cpu_baseline"] = {"value": n / sec, "unit": "queries/s", "cores": blas_threads(),
                                "kind": "oracle",
                                "sample": f"{n} BetaE queries (1 per type), literal-KL scoring "
                                          f"over all 14,505 entities + full sort, float64 numpy"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def secondary_passes(args, t, groups, mixed_mode, flush):
    """One GPU: (1) the step form the headline did not use -- the 14 per-type submits over 3
    streams, or one mixed submit; (2) every query type alone (one kgq_submit of its 1024 queries,
    nothing else on the GPU): the metric's "queries/sec per query type"."""
    import torch
    from paper_2503_02172_b200 import Engine
    qs = {g[0]: (torch.from_numpy(g[2]).cuda(), torch.from_numpy(g[3]).cuda()) for g in groups}
    main = torch.cuda.current_stream()

    def time_fn(fn, n):
        ms = 0.0
        for _ in range(n):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main)
            fn()
            e1.record(main)
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
        return ms / n

    S = 3
    engs = []
    for _ in range(S):
        e = Engine("betae", N_ENT, N_REL, DIM, hidden=HID, max_batch=BATCH, max_k=K)
        e.load_tables(t)
        engs.append(e)
    out = {s: (torch.empty((BATCH, K), device="cuda"), torch.empty((BATCH, K), dtype=torch.int32, device="cuda"))
           for s in STRUCTS}
    per_type = {}
    for s in STRUCTS:
        fn = lambda s=s: engs[0].submit(s, *qs[s], K, out=out[s], stream=main)
        for _ in range(3):
            fn()
        per_type[s] = BATCH / (time_fn(fn, args.steps) / 1e3)
    per_type_info = {"qps": per_type, "how": "each type alone: one kgq_submit of its 1024 queries on one stream, "
                                             "L2 flushed before each (device time)"}
    if mixed_mode:
        streams = [torch.cuda.Stream() for _ in range(S)]

        def fork_join():
            ev0 = torch.cuda.Event()
            ev0.record(main)
            for st in streams:
                st.wait_event(ev0)
            for i, s in enumerate(STRUCTS):
                engs[i % S].submit(s, *qs[s], K, out=out[s], stream=streams[i % S])
            for st in streams:
                ev = torch.cuda.Event()
                ev.record(st)
                main.wait_event(ev)
        for _ in range(3):
            fork_join()
        ms = time_fn(fork_join, args.steps)
        other = {"form": f"the 14 per-type kgq_submit calls over {S} streams (one context each)",
                 "value": len(STRUCTS) * BATCH / (ms / 1e3), "ms_per_step": ms}
    else:
        meng = Engine("betae", N_ENT, N_REL, DIM, hidden=HID, max_batch=BATCH * len(STRUCTS), max_k=K)
        meng.load_tables(t)
        a = torch.from_numpy(np.concatenate([g[2].reshape(-1) for g in groups])).cuda()
        r = torch.from_numpy(np.concatenate([g[3].reshape(-1) for g in groups])).cuda()
        mo = (torch.empty((BATCH * len(STRUCTS), K), device="cuda"),
              torch.empty((BATCH * len(STRUCTS), K), dtype=torch.int32, device="cuda"))
        fn = lambda: meng.submit_mixed_packed([g[0] for g in groups], [g[1] for g in groups], a, r, K, mo, stream=main)
        for _ in range(3):
            fn()
        ms = time_fn(fn, args.steps)
        meng.check_errors()
        meng.close()
        other = {"form": "one kgq_submit_mixed of the 14 x 1024 queries", "value": len(STRUCTS) * BATCH / (ms / 1e3),
                 "ms_per_step": ms}
    for e in engs:
        e.check_errors()
        e.close()
    return other, per_type_info


if __name__ == "__main__":
    main()
