#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/r02_uv_ab.txt
: > $O
for lib in paper_2503_02172_b200/libkgq.so ab_libs/libkgq_m3u4.so ab_libs/libkgq_m3u8.so ab_libs/libkgq_m2u12.so; do
  echo "== $lib" >> $O
  KGQ_LIB_PATH=$PWD/$lib timeout 300 python bench.py --workload c5a --models betae --steps 5 --warmup 2 >> $O 2>&1
done
bash scripts/gpu.sh multirank suite
