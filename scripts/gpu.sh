#!/bin/bash
# GPU-box recipes (run through gpurun from the repo root):
#   gpurun -- 'bash scripts/gpu.sh TASK [TASK ...]'
# Tasks (outputs under gpurun_out/, which gpurun brings back):
#   smoke      __graft_entry__.smoke()
#   tests      pytest -m gpu (all GPU parity tests)
#   bench      default bench.py line (C2 headline + e2e + mixed + C5a HBM + cpu_baseline)
#   reference  bench.py --impl reference (the oracle arm)
#   suite      bench.py --workload suite (the other BASELINE configs)
#   launches   ncu launch list of one bench step (gpu__time_duration, DRAM bytes per launch)
#   launches-warm  the same launch list with warm caches (--cache-control none)
#   ncu-small  ncu --set full of one mixed step's small kernels (gather / scatter / combine / score prep / top-k)
#   ncu-score  ncu --set full of the two BetaE scorer launches of one mixed step
#   quick      the default bench line without the side measurements (one summary line)
#   ncu-gemm   ncu --set full of k_gemm launches of one bench step (a dense layer + the scorer)
#   ncu-c5a    ncu --set full of the C5a streaming scorer (GQE 1p, B = 8)
#   sanitize   compute-sanitizer memcheck / racecheck / synccheck on small configs
#   chain      per-structure chain / full-row distance errors (scripts/diag_chain_err.py)
#   ab         same-box A/B of the in-tree libkgq.so vs ab_libs/$AB_LIB on the C2 bench
#   streams    the headline step over 1-4 streams, and with the GEMM grid capped (KGQ_GEMM_CLUSTERS)
#   multirank  the N > 1 bench path with both ranks on the one GPU (gloo; a path check, numbers meaningless)
#   probes     tcgen05 GEMM checker / throughput probe / MMA issue probe (built by scripts/tc_probe.sh)
#   accuracy   chain / whole-row distance errors vs the oracle for both operand builds (fp16x2 libkgq.so,
#              bf16x3 libkgq_bf16x3.so) on the small, spread, medium, C2 and C4 configs
#   raster-ab  the headline step with the GEMM tile raster group at 0 (M fastest) / 4 / 8 / 16
#   fp32-pipe  FP32 issue-rate probe (FADD / FFMA / FADD2 / FFMA2 / FMNMX lane-ops per clock)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OUT=gpurun_out
for task in "$@"; do
  echo "== $task"
  case "$task" in
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1; tail -2 $OUT/smoke.txt ;;
    tests) timeout 1800 python -m pytest tests -m gpu -q -rs --durations=15 > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt; tail -3 $OUT/pytest_gpu.txt ;;
    bench) timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; tail -2 $OUT/bench.err ;;
    reference) timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err ;;
    suite) timeout 1500 python bench.py --workload suite --steps 5 --warmup 2 > $OUT/suite.jsonl 2> $OUT/suite.err ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
                --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-mixed --no-c5a > /dev/null 2>&1 ;;
    launches-warm) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
                --cache-control none --csv --log-file $OUT/launches_warm.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
                --no-per-type --no-c5a > /dev/null 2>&1 ;;
    ncu-small) timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mix_score_prep|k_mix_gather|k_topk_cmin|k_topk_lists|k_mix_scatter|k_mix_combine|k_mix_h0_pre" \
                -s 11 -c 11 -o $OUT/prof_small -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-per-type --no-c5a > /dev/null 2>&1 ;;
    ncu-score) timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiBetaScore -s 2 -c 2 \
                -o $OUT/prof_score -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-per-type --no-c5a > /dev/null 2>&1 ;;
    quick) timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-per-type --no-c5a > $OUT/quick.json 2> $OUT/quick.err
           python -c "import json; d=json.load(open('$OUT/quick.json')); p=d['roofline']['parts']; print('quick', round(d['value']), round(d['ms_per_step'], 3), 'dense', round(p['dense']['tflops'], 1), 'score', round(p['score']['tflops'], 1), p['score']['ms_per_step'])" ;;
    ncu-gemm) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 30 -c 4 -o $OUT/prof_gemm -f \
                python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-mixed --no-c5a --streams 1 > /dev/null 2>&1 ;;
    ncu-c5a) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_score_stream -s 2 -c 1 -o $OUT/prof_c5a -f \
               python scripts/c5a_one.py gqe 1p 8 3 > /dev/null 2>&1
             timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_score_uv_stream -s 2 -c 1 -o $OUT/prof_c5a_betae -f \
               python scripts/c5a_one.py betae 2u 8 3 > /dev/null 2>&1 ;;
    sanitize) bash scripts/sanitize.sh > $OUT/sanitize.txt 2>&1; tail -12 $OUT/sanitize.txt ;;
    chain) timeout 900 python scripts/diag_chain_err.py small medium c2 c4 > $OUT/chain_err.jsonl 2>&1 ;;
    ab) for i in 1 2; do
          for lib in paper_2503_02172_b200/libkgq.so ab_libs/${AB_LIB:-libkgq_prev.so}; do
            KGQ_LIB_PATH=$PWD/$lib timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-mixed --no-c5a \
              > $OUT/ab.json 2> $OUT/ab.err || tail -3 $OUT/ab.err
            python -c "import json; d=json.load(open('$OUT/ab.json')); print('$lib', round(d['value']), round(d['ms_per_step'], 3), d['sequential'])" | tee -a $OUT/ab.txt
          done
        done ;;
    streams) for S in 1 2 3 4; do timeout 900 python bench.py --steps 10 --warmup 3 --streams $S --no-cpu-baseline --no-mixed --no-c5a \
               > $OUT/streams_$S.json 2> $OUT/streams_$S.err; done
             for C in 56 48 37; do KGQ_GEMM_CLUSTERS=$C timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-mixed \
               --no-c5a > $OUT/clusters_$C.json 2> $OUT/clusters_$C.err; done ;;
    multirank) KGQ_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
                 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --no-c5a --no-mixed > $OUT/multirank.json 2> $OUT/multirank.err
               tail -3 $OUT/multirank.err ;;
    probes) ( cd scripts; timeout 120 ./tc_bn_check; timeout 200 ./tc_probe_base; timeout 120 ./mma3_probe ) > $OUT/probes.txt 2>&1 ;;
    accuracy) for lib in libkgq.so libkgq_bf16x3.so; do echo "== $lib"
                KGQ_LIB_PATH=$PWD/paper_2503_02172_b200/$lib timeout 900 python scripts/diag_chain_err.py small small_spread \
                  medium c2 c4 2>&1 | tail -5
              done > $OUT/accuracy.jsonl ;;
    raster-ab) for g in 0 4 8 16; do KGQ_GEMM_GROUP_M=$g bash "$0" quick | grep "^quick [0-9]" | sed "s/^/group_m $g /"; done \
                 | tee $OUT/raster_ab.txt ;;
    fp32-pipe) ( cd scripts; /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_pipe_probe \
                 fp32_pipe_probe.cu && timeout 120 ./fp32_pipe_probe ) > $OUT/fp32_pipe.txt 2>&1 ;;
    *) echo "unknown task $task" ;;
  esac
done
ls $OUT
