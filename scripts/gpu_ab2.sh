cd $GRAFT_REPO_ROOT
for env in "X=1" "KGQ_NO_SPLITK=1"; do
  env $env timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:k_gemm --csv --log-file gpurun_out/ab_$(echo $env | cut -c1-5).csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
ls gpurun_out
