#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 ./scripts/mma3_probe > gpurun_out/r02_mma3_probe.txt 2>&1
echo "rc=$?" >> gpurun_out/r02_mma3_probe.txt
timeout 900 python -m pytest tests -m gpu -q -rs -k "softmax or peer or nccl or comm" > gpurun_out/r02_pytest_gpu2.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu2.txt
