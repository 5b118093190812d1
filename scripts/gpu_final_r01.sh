# round-1 evidence: default bench line (with cpu_baseline), reference arm, suite, C5a latency,
# ncu launch list of one bench step and a --set full capture of the dominant GEMM launches
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -2 gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --workload suite --steps 5 --warmup 2 > gpurun_out/suite_final.jsonl 2> gpurun_out/suite_final.err
timeout 900 python bench.py --workload c5a --steps 10 --warmup 3 > gpurun_out/c5a_final.json 2> gpurun_out/c5a_final.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-mixed > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 3 -c 4 -o gpurun_out/prof_gemm_final python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-mixed > /dev/null 2>&1
ls -la gpurun_out
