#!/bin/bash
# fp16x2 operands: chain / distance errors vs the oracle (scripts/diag_chain_err.py) and the mixed
# step for DRAIN 4 (in-tree), 8 and 16 (ab_libs builds).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in paper_2503_02172_b200/libkgq.so ab_libs/libkgq_d8.so ab_libs/libkgq_d16.so; do
  echo "== $lib"
  KGQ_LIB_PATH=$PWD/$lib timeout 900 python scripts/diag_chain_err.py small small_spread medium c2 c4 2>&1 | tail -5
  KGQ_LIB_PATH=$PWD/$lib bash scripts/gpu.sh quick | grep "^quick [0-9]"
done
