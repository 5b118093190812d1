# A/B of env switches on the C2 bench (device-timed value and stage split)
cd $GRAFT_REPO_ROOT
for env in ${AB_ENVS:-"X=1" "KGQ_NO_SPLITK=1"}; do
  env $env timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$env', round(d['value']), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms_per_step'].items()})
"
done
