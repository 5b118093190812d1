#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/r02_uv_ab3.txt
: > $O
timeout 900 python -m pytest tests -m gpu -q -x -k "extremes or 2m or toy or edge or max_batch or every_structure or softmax or concurrent or ktime" >> $O 2>&1
timeout 300 python bench.py --workload c5a --models betae --steps 5 --warmup 2 >> $O 2>&1
