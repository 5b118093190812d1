# launch list of one bench step + ncu --set full of the dominant kernels (score GEMM, MLP GEMM)
cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 3 -c 4 -o gpurun_out/prof_gemm_r01b python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
