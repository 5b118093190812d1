#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "extremes or 2m or toy or edge or planted or max_batch" > gpurun_out/r02_pytest_c5a.txt 2>&1
echo "rc=$?" >> gpurun_out/r02_pytest_c5a.txt
timeout 600 python bench.py --workload c5a --steps 5 --warmup 2 > gpurun_out/r02_c5a_tma.json 2>&1
KGQ_SCORE_STREAM=regs timeout 600 python bench.py --workload c5a --steps 5 --warmup 2 > gpurun_out/r02_c5a_regs.json 2>&1
