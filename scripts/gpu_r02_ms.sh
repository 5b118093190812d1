#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/multistream_probe.py 1 2 3 4 > gpurun_out/r02_multistream.jsonl 2>&1
KGQ_PDL=0 timeout 300 python scripts/multistream_probe.py 1 2 3 4 >> gpurun_out/r02_multistream.jsonl 2>&1
KGQ_PDL_SMALL=1 timeout 300 python scripts/multistream_probe.py 1 2 4 >> gpurun_out/r02_multistream.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/r02_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu.txt
