# Same-box A/B of two library builds on the C2 bench: current in-tree libkgq.so vs ab_libs/$AB_LIB
cd $GRAFT_REPO_ROOT
for i in 1 2; do
  for lib in paper_2503_02172_b200/libkgq.so ab_libs/${AB_LIB:-libkgq_prev.so}; do
    KGQ_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-mixed > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$lib', round(d['value']), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms_per_step'].items()})
"
  done
done
