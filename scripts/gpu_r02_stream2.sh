#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/r02_stream_ab2.txt
: > $O
timeout 600 python -m pytest tests -m gpu -q -x -k "extremes or 2m or toy or edge or max_batch or every_structure or softmax" >> $O 2>&1
for lib in paper_2503_02172_b200/libkgq.so ab_libs/libkgq_uv2.so ab_libs/libkgq_uv8.so; do
  echo "== $lib" >> $O
  KGQ_LIB_PATH=$PWD/$lib timeout 300 python bench.py --workload c5a --models betae --steps 5 --warmup 2 >> $O 2>&1
done
echo "== gqe default" >> $O
timeout 300 python bench.py --workload c5a --models gqe --steps 5 --warmup 2 >> $O 2>&1
