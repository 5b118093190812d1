#!/usr/bin/env python
"""Benchmark of the CLQA inference hot path (BASELINE.json metric).

Workload (N=1): BASELINE.json configs[1] -- BetaE on the synthetic FB15k-237 shape
(14,505 entities, 237 relations, d 400, MLP 1600x2), batch 1024, all 14 query types.
One step = one batch of every query type through the whole path (operator chain ->
entity scoring -> top-k 10), i.e. 14 x 1024 queries.  value = queries/s over all ranks.

N > 1 (torchrun): the entity table is sharded over the ranks; queries are
replicated; each rank returns its local top-k, an NCCL all-gather exchanges them and
kgq_merge_topk merges -> strong scaling of the same workload.

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
    fp32 FLOPs vs the bf16x3 peak = measured bf16 / 6)."""
    import torch
    from paper_2503_02172_b200 import Engine
    peaks, src = load_peaks()
    alu_peak = 148 * 128 * peaks.get("sm_max_mhz", 1965.0) * 1e6  # lane-instr/s
    tc_peak = peaks["bf16_tflops"] / 6.0
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
        tot = sum(per.values())
        q = args.steps * len(structs) * B
        st = {k: v[0] / args.steps for k, v in prof.items()}
        sc_ms, _, sc_w = prof["score"]
        d_ms, _, d_w = prof["dense"]
        if model == "betae" and B > 16:
            ach = (sc_w + d_w) / ((sc_ms + d_ms) / 1e3) / 1e12
            roof = {"kernel": "k_gemm (tcgen05 bf16x3: dense layers + BetaE scorer)", "bound": "tensor",
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
                          "l2": "flushed between steps"}), flush=True)


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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kgq", choices=["kgq", "reference"])
    ap.add_argument("--streams", type=int, default=3,
                    help="concurrent streams per GPU (one library context each); the 14 per-type submits of a "
                         "step are dealt round-robin over them")
    ap.add_argument("--split", default="queries", choices=["queries", "entities"],
                    help="N>1: rank r runs rows [r B, (r+1) B) of a W x B replicated batch (weak scaling, the "
                         "library's query-split communicator), or the entity table is sharded over the ranks "
                         "with a replicated B-query batch (strong scaling, local top-k + all-gather + merge)")
    ap.add_argument("--merge", default="nccl", choices=["nccl", "p2p", "torch"],
                    help="entity split: the library's NCCL all-gather + merge kernel (default), the all-gather "
                         "fused into the top-k over symmetric peer memory (N2), or torch.distributed + merge")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-queries", type=int, default=14)
    ap.add_argument("--no-mixed", action="store_true", help="skip the mixed-structure submit measurement")
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
    S = max(1, args.streams)
    # the query split runs through the library's NCCL communicator, which needs one GPU per rank:
    # the one-GPU path check uses the entity split with the torch.distributed merge instead
    qsplit = world > 1 and args.split == "queries" and not one_gpu
    # per-type batch of the replicated input: W x 1024 in query split (each rank runs 1024 rows:
    # weak scaling), else 1024 (entity split: strong scaling over the entity table)
    Bg = BATCH * world if qsplit else BATCH
    merge = "nccl" if qsplit else (args.merge if not one_gpu else "torch")
    t = synth.make_tables("betae", N_ENT, N_REL, DIM, hidden=HID, seed=SEED)
    engines = []
    for _ in range(S):
        se = ShardedEngine("betae", N_ENT, N_REL, DIM, split="queries" if qsplit else "entities", hidden=HID,
                           max_batch=Bg, max_k=K, device=local, merge=merge)
        se.load_tables(t)
        se.p2p_check = False  # N2 errors are checked once after the timed steps
        se.engine.ktime(True)  # in-kernel GEMM launch spans (roofline from this very pass)
        engines.append(se)
    streams = [torch.cuda.Stream() for _ in range(S)]
    main_stream = torch.cuda.current_stream()
    qs = {}
    for s in STRUCTS:
        if qsplit:  # the same per-rank 1024-query batches as N = 1, replicated over all ranks
            parts = [synth.make_queries(s, BATCH, N_ENT, N_REL, seed=synth.query_seed(SEED, s) + 7919 * w)
                     for w in range(world)]
            a, r = np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])
        else:
            a, r = synth.make_queries(s, BATCH, N_ENT, N_REL, seed=synth.query_seed(SEED, s))
        qs[s] = (a, r, torch.from_numpy(a).cuda(), torch.from_numpy(r).cuda())
    outs = {s: (torch.empty((Bg, K), device="cuda"), torch.empty((Bg, K), dtype=torch.int32, device="cuda"))
            for s in STRUCTS}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    launches = [0]
    lane = {s: i % S for i, s in enumerate(STRUCTS)}

    def step(nlanes=S, count=True):
        """One step: the 14 per-type submits dealt over `nlanes` streams, joined on the main
        stream; returns the (start, end) events of the main stream."""
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(main_stream)
        for st in streams[:nlanes]:
            st.wait_event(e0)
        for s in STRUCTS:
            j = lane[s] % nlanes
            engines[j].submit(s, qs[s][2], qs[s][3], K, stream=streams[j])
            if count:
                launches[0] += engines[j].last_launch_count()
        for st in streams[:nlanes]:
            ev = torch.cuda.Event()
            ev.record(st)
            main_stream.wait_event(ev)
        e1.record(main_stream)
        return e0, e1

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(nsteps, nlanes):
        """nsteps steps, L2 flushed (untimed) before each; per-step device ms (start event on
        the main stream before the fork, end event after every stream joined)."""
        ms = []
        for _ in range(nsteps):
            flush.zero_()
            e0, e1 = step(nlanes)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return ms

    for _ in range(args.warmup):
        step(S, False)
        step(1, False)  # the sequential pass's graphs (lane 0) are captured here too
    barrier()
    for se in engines:
        se.engine.check_errors()
        se.engine.ktime_read()
        se.engine.ktime_log()
    launches[0] = 0
    with ClockSampler(local) as clk:
        barrier()
        step_ms = timed(args.steps, S)
        barrier()
    n_launch = launches[0]
    # GEMM launch spans of exactly these steps (every context's log, one clock per device)
    logs = [se.engine.ktime_log() for se in engines]
    kt = [se.engine.ktime_read() for se in engines]
    spans = np.concatenate([lg for lg in logs if len(lg)]) if any(len(lg) for lg in logs) else np.zeros((0, 3), np.uint64)
    gemm_busy_ms = span_union_ms(spans[:, :2]) / args.steps
    dense_busy_ms = span_union_ms(spans[spans[:, 2] == 0][:, :2]) / args.steps
    score_busy_ms = span_union_ms(spans[spans[:, 2] == 1][:, :2]) / args.steps
    dense_span_sum = sum(k["dense"][0] for k in kt) / args.steps
    score_span_sum = sum(k["score"][0] for k in kt) / args.steps
    gemm_launches = sum(k["dense"][1] + k["score"][1] for k in kt) / args.steps
    total_ms = sum(step_ms)
    # sequential reference pass: the same steps on ONE stream (round-1's headline form)
    seq_ms = None
    seq_dense_ms = seq_score_ms = None
    if S > 1:
        barrier()
        seq = timed(args.steps, 1)
        seq_ms = sum(seq)
        lg = engines[0].engine.ktime_log()  # one stream: every GEMM alone on the GPU
        seq_dense_ms = span_union_ms(lg[lg[:, 2] == 0][:, :2]) / args.steps
        seq_score_ms = span_union_ms(lg[lg[:, 2] == 1][:, :2]) / args.steps
        for se in engines:
            se.engine.ktime_log()
            se.engine.ktime_read()
    if world > 1:
        tt = torch.tensor([total_ms, seq_ms or 0.0], dtype=torch.float64, device="cuda" if not one_gpu else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms, seq_ms = float(tt[0].item()), (float(tt[1].item()) or None)
    per_rank_queries = len(STRUCTS) * BATCH  # per step (query split: each rank's own rows)
    job_queries = per_rank_queries * (world if qsplit else 1)
    value = job_queries * args.steps / (total_ms / 1e3)

    # ---- algorithmic GEMM FLOPs per step (the library's own work counters, one profiled
    # submit per type outside the timed region) ----
    eng0 = engines[0].engine
    eng0.ktime(False)
    eng0.profile(True)
    eng0.profile_read()
    for s in STRUCTS:
        engines[0].submit(s, qs[s][2], qs[s][3], K)
    torch.cuda.synchronize()
    prof = eng0.profile_read()
    eng0.profile(False)
    d_fl, s_fl = prof["dense"][2], prof["score"][2]  # query split: this rank's rows (per-GPU FLOPs)

    # ---- the same step as ONE mixed-structure submit (kgq_submit_mixed) ----
    mixed = None
    if world == 1 and not args.no_mixed:
        meng = Engine("betae", N_ENT, N_REL, DIM, hidden=HID, max_batch=BATCH * len(STRUCTS), max_k=K, device=local)
        meng.load_tables(t)
        groups = [(s, qs[s][2].int(), qs[s][3].int()) for s in STRUCTS]
        mout = (torch.empty((BATCH * len(STRUCTS), K), device="cuda"),
                torch.empty((BATCH * len(STRUCTS), K), dtype=torch.int32, device="cuda"))
        for _ in range(args.warmup):
            meng.submit_mixed(groups, K, out=mout)
        torch.cuda.synchronize()
        meng.check_errors()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        mt = 0.0
        for _ in range(args.steps):
            flush.zero_()
            e0.record()
            meng.submit_mixed(groups, K, out=mout)
            e1.record()
            torch.cuda.synchronize()
            mt += e0.elapsed_time(e1)
        mixed = {"value": per_rank_queries * args.steps / (mt / 1e3), "unit": "queries/s",
                 "ms_per_step": mt / args.steps,
                 "how": "one kgq_submit_mixed per step with the same 14 x 1024 queries on one stream (L2 flushed "
                        "between steps): each projection hop of all 14 types' branches is one MLP"}
        meng.close()

    # ---- end to end through the public API with host buffers (pinned), same streams ----
    pin = {s: (torch.from_numpy(qs[s][0]).pin_memory(), torch.from_numpy(qs[s][1]).pin_memory()) for s in STRUCTS}
    hout = {s: (torch.empty((Bg, K)).pin_memory(), torch.empty((Bg, K), dtype=torch.int32).pin_memory())
            for s in STRUCTS}
    h2d = sum(Bg * (qs[s][0].shape[1] + qs[s][1].shape[1]) * 4 for s in STRUCTS)
    d2h = len(STRUCTS) * Bg * K * 8
    e2e_v = None
    try:
        def e2e_step():
            for s in STRUCTS:
                j = lane[s]
                engines[j].engine.submit_host(s, pin[s][0].numpy(), pin[s][1].numpy(), K,
                                              out=(hout[s][0].numpy(), hout[s][1].numpy()), stream=streams[j],
                                              sync=False)
            for st in streams:
                st.synchronize()
        e2e_step()
        e2e_step()
        e2e_s = 0.0
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            t0 = time.perf_counter()
            e2e_step()
            e2e_s += time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([e2e_s], dtype=torch.float64, device="cuda" if not one_gpu else "cpu")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt.item())
        e2e_v = job_queries * args.steps / e2e_s
    except Exception as ex:  # a failure here must not cost the headline line: e2e is then null
        print(f"bench: e2e failed: {type(ex).__name__}: {ex}", file=sys.stderr, flush=True)
    for se in engines:
        se.engine.check_errors()

    # ---- C5a: the north-star HBM target (2M-entity scoring sweep, B in {1, 8}) ----
    peaks, peak_src = load_peaks()
    c5a = None
    if world == 1 and not args.no_c5a:
        try:
            c5a = c5a_measure(max(3, args.steps // 2), 2, peaks)
        except Exception as ex:
            print(f"bench: C5a failed: {type(ex).__name__}: {ex}", file=sys.stderr, flush=True)

    # ---- roofline of the dominant kernel: the tcgen05 bf16x3 GEMM (k_gemm), which runs every
    # dense layer of the chain and the BetaE scorer contraction.  Algorithmic work = useful fp32
    # FLOPs (2MNK, the library's counters); time = the union of the GEMM launches' in-kernel spans
    # (%globaltimer, first CTA start after the PDL wait -> last CTA end) over the timed steps of
    # THIS pass, merged over the concurrent streams; peak = measured bf16 / 6 (six bf16 MMAs per
    # useful fp32 multiply-add: x0w0, x0w1, x1w0, x0w2, x1w1, x2w0), the BURST figure: the
    # scorer GEMM alone measures above the driver's sustained (4-s cuBLAS loop under the power
    # cap) figure in this duty cycle, so only the burst one is a ceiling; the sustained fraction
    # is quoted beside it.
    peak_sus = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) / 6.0
    peak_burst = peaks["bf16_tflops"] / 6.0
    rate = lambda fl, ms: fl / (ms / 1e3) / 1e12 if ms > 0 else 0.0
    achieved = rate(d_fl + s_fl, gemm_busy_ms)
    traffic = None
    tf = os.path.join(ROOT, "profiles", "tc_gemm_traffic.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get("dram_bytes_per_launch")
    if rank == 0:
        ms_step = total_ms / args.steps
        line = {
            "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak" if qsplit or world == 1 else "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(CONFIG, l2="flushed between timed steps (256 MiB write, untimed)",
                           streams=S,
                           parallelism=("1 GPU" if world == 1 else
                                        f"query split x{world} (W x 1024 replicated rows per type, each rank its "
                                        f"1024; library NCCL all-gather)" if qsplit else
                                        f"entity shards x{world} ({engines[0].merge_mode})"),
                           batch_per_type=Bg),
            "how": (f"per step: the 14 per-type kgq_submit calls (1024 queries each per rank) dealt round-robin over "
                    f"{S} CUDA streams, one library context per stream; device time from an event before the "
                    f"fork to an event after the join, max over ranks"),
            "sequential": None if seq_ms is None else {
                "value": job_queries * args.steps / (seq_ms / 1e3), "ms_per_step": seq_ms / args.steps,
                "how": "the same steps with the 14 submits on one stream (no overlap between types)"},
            "gemm": {"busy_ms_per_step": gemm_busy_ms, "dense_busy_ms_per_step": dense_busy_ms,
                     "score_busy_ms_per_step": score_busy_ms, "dense_span_sum_ms": dense_span_sum,
                     "score_span_sum_ms": score_span_sum, "launches_per_step": gemm_launches,
                     "share_of_step": gemm_busy_ms / ms_step,
                     "how": "in-kernel %globaltimer spans of every k_gemm launch of the timed steps (kgq_ktime_log), "
                            "union over the concurrent streams"},
            "roofline": {"kernel": "k_gemm (tcgen05 bf16x3: chain dense layers + BetaE scorer)",
                         "bound": "tensor", "achieved": achieved, "peak": peak_burst, "unit": "TFLOP/s",
                         "frac": achieved / peak_burst, "traffic": traffic,
                         "peak_source": f"{peak_src} bf16 burst {peak_burst * 6:.1f} / 6 (bf16x3: 6 MMAs per fp32 MAC)",
                         "frac_vs_sustained": achieved / peak_sus,
                         "work": f"useful fp32 FLOPs 2MNK per GEMM launch: {(d_fl + s_fl) / 1e9:.1f} GFLOP per step "
                                 f"per rank (dense {d_fl / 1e9:.1f}, score {s_fl / 1e9:.1f})",
                         "whole_step_rate": rate(d_fl + s_fl, ms_step),
                         "parts": None if seq_dense_ms is None else {
                             "how": "each part's GEMMs alone on the GPU: the sequential (one-stream) pass's in-kernel "
                                    "spans; under the concurrent streams the parts overlap each other",
                             "dense": {"ms_per_step": seq_dense_ms, "tflops": rate(d_fl, seq_dense_ms),
                                       "frac": rate(d_fl, seq_dense_ms) / peak_burst},
                             "score": {"ms_per_step": seq_score_ms, "tflops": rate(s_fl, seq_score_ms),
                                       "frac": rate(s_fl, seq_score_ms) / peak_burst}}},
            "gpu_launches": n_launch,
            "mixed_submit": mixed,
            "e2e": {"value": e2e_v, "unit": "queries/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "how": (f"per step: kgq_submit_host_async per type on the same {S} streams (pinned H2D of "
                            f"anchors / relations, path, D2H of the top-k into pinned host outputs), every stream "
                            f"synchronised; wall clock, L2 flushed before each step (untimed), max over ranks")},
            "hbm": None if c5a is None else {
                "workload": "BASELINE.json configs[4] latency regime: 2M entities, d 400, 1 GPU, GQE / BetaE, "
                            "1p / 2u, B in {1, 8}",
                "kernel": "k_score_stream (streaming entity scorer)", "bound": "hbm", "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "peak_source": f"{peak_src} copy bandwidth",
                "work": "the shard's scoring table read once per batch: GQE 4 N d bytes, BetaE 8 N d (the centred "
                        "fp32 u, v planes)",
                "alu_peak": "148 SMs x 128 FP32 lanes x max SM clock (FFMA2 / FADD counted per lane operation)",
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


if __name__ == "__main__":
    main()
