cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_topk -s 3 -c 1 -o gpurun_out/prof_topk5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out | grep topk5
