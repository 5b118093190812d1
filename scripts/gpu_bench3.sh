cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -3 gpurun_out/bench3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 20 -c 6 -o gpurun_out/prof_tc3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_topk -s 3 -c 1 -o gpurun_out/prof_topk3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
