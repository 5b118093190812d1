cd $GRAFT_REPO_ROOT
timeout 60 ./scripts/tc_perf_base 2>&1 | grep "BN=  0"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
for k in ['value','ms_per_step','stage_ms_per_step','roofline','clocks']: print(k, d[k])
"
