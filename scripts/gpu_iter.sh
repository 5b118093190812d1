# probe + parity + C2 bench: the per-change GPU check of the GEMM core
cd $GRAFT_REPO_ROOT
bash scripts/tc_probe.sh run 2>&1 | tee gpurun_out/tc_probe.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x 2>&1 | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
for k in ['value','ms_per_step','stage_ms_per_step','roofline','clocks','e2e']: print(k, d.get(k))
"
