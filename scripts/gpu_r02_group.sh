#!/bin/bash
# A/B of the GEMM tile raster (KGQ_GEMM_GROUP_M: 0 = M fastest, else M blocks per group) on the
# default (mixed) bench step, two rounds, same box.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rnd in 1 2; do
  for g in ${GM_LIST:-0 4 8 16}; do
    KGQ_GEMM_GROUP_M=$g timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-per-type --no-c5a \
      > gpurun_out/group_$g.json 2> gpurun_out/group_$g.err || tail -3 gpurun_out/group_$g.err
    python -c "import json; d=json.load(open('gpurun_out/group_$g.json')); p=d['roofline']['parts']; print('group_m $g', round(d['value']), round(d['ms_per_step'],3), 'dense', round(p['dense']['tflops'],1), 'score', round(p['score']['tflops'],1), 'e2e', round(d['e2e']['value']))" | tee -a gpurun_out/group_ab.txt
  done
done
