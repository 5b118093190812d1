# parity + fullsize + C2 bench (+ C5a latency bench): the per-change GPU check
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
for k in ['value','ms_per_step','stage_ms_per_step','roofline','clocks','e2e']: print(k, d.get(k))
"
timeout 600 python bench.py --workload c5a --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c5a.json 2> gpurun_out/c5a.err; tail -3 gpurun_out/c5a.err
python -c "
import json; d=json.load(open('gpurun_out/c5a.json'))
for k in ['value','unit','ms_per_step','latency','roofline']: print(k, d.get(k))
"
