#!/bin/bash
# Round-2 evidence for the docs: default bench line, reference arm, multi-rank path check,
# ncu launch list (cold and warm) of one headline step, ncu --set full of the scorer and the
# largest dense layer.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OUT=gpurun_out
bash scripts/gpu.sh smoke bench reference multirank
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-per-type --no-c5a > /dev/null 2>&1
bash scripts/gpu.sh launches-warm
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiBetaScore \
  -s 2 -c 2 -o $OUT/prof_score -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-per-type --no-c5a > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 17 -c 2 -o $OUT/prof_dense -f \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-per-type --no-c5a > /dev/null 2>&1
ls $OUT
