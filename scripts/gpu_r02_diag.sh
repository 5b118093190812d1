#!/bin/bash
# round-2 diagnostics: chain / full-row distance errors for DRAIN 8 / 4 / 2 builds, plus the headline bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_smi.txt
python scripts/diag_chain_err.py small medium c2 c4 > gpurun_out/r02_chain_d8.jsonl 2>&1
KGQ_LIB_PATH=$PWD/ab_libs/libkgq_d4.so python scripts/diag_chain_err.py small medium c2 c4 > gpurun_out/r02_chain_d4.jsonl 2>&1
KGQ_LIB_PATH=$PWD/ab_libs/libkgq_d2.so python scripts/diag_chain_err.py small medium c2 c4 > gpurun_out/r02_chain_d2.jsonl 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_d8.json 2>gpurun_out/r02_bench_d8.err
KGQ_LIB_PATH=$PWD/ab_libs/libkgq_d4.so python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_d4.json 2>gpurun_out/r02_bench_d4.err
KGQ_LIB_PATH=$PWD/ab_libs/libkgq_d2.so python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_d2.json 2>gpurun_out/r02_bench_d2.err
