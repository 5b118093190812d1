#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -k "ktime" > gpurun_out/r02_pytest_ktime.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench_v1.json 2> gpurun_out/r02_bench_v1.err
timeout 600 ncu --set full --clock-control none -k regex:k_score_stream -s 2 -c 1 -o gpurun_out/r02_c5a_gqe_b8 -f python scripts/c5a_one.py gqe 1p 8 3 > gpurun_out/r02_ncu_c5a.log 2>&1
