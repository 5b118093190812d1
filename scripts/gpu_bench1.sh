set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-queries 2 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err
cat gpurun_out/bench1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
wc -l gpurun_out/launches1.csv
