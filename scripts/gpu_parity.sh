set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -30
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu 2>&1 | tail -15
