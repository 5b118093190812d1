#!/bin/bash
# round 2: full GPU test suite + chain diagnostics of the spread / GQE / Q2B configs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -rs --durations=15 > gpurun_out/r02_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu.txt
timeout 600 python scripts/diag_chain_err.py small_spread gqe_spread q2b_spread gqe_small q2b_small c3 > gpurun_out/r02_chain_more.jsonl 2>&1
