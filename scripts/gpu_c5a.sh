cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --workload c5a --steps 10 --warmup 3 > gpurun_out/c5a.json 2> gpurun_out/c5a.err; tail -3 gpurun_out/c5a.err
cat gpurun_out/c5a.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c5a_launches.csv python bench.py --workload c5a --steps 1 --warmup 1 > /dev/null 2>&1
