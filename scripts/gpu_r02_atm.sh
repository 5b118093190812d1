#!/bin/bash
# round 2: A-operand-in-TMEM probe (correctness + throughput) and the GPU test suite
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( cd scripts; echo "== bn check (A in TMEM)"; timeout 120 ./tc_bn_check_atm; echo "rc=$?"
  echo "== bn check (base)"; timeout 120 ./tc_bn_check | tail -2
  echo "== probe base"; timeout 200 ./tc_probe_base; echo "== probe A in TMEM"; timeout 200 ./tc_probe_atm ) > gpurun_out/r02_atm_probe.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/r02_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu.txt
