# bf16x3 GEMM: tile-width/epilogue check vs fp64, probe, parity, C2 bench
cd $GRAFT_REPO_ROOT/scripts
timeout 120 ./tc_bn_check 2>&1 | tail -25
timeout 120 ./tc_probe_base 2>&1
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -15
AB_ENVS="X=1" bash scripts/gpu_ab.sh
