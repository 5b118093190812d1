# Build (here, CPU) or run (GPU box: `run`) the persistent tc GEMM probe and its checkers.
cd "$(dirname "$0")"
NVCC=/usr/local/cuda/bin/nvcc
FL="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -lcuda -diag-suppress 177"
if [ "$1" = "run" ]; then
  echo "== bn check"; timeout 120 ./tc_bn_check
  echo "== probe"; timeout 120 ./tc_probe_base
  echo "== probe (PDL)"; KGQ_PDL=1 timeout 120 ./tc_probe_base
  echo "== trace"; timeout 120 ./tc_probe_trace
  for v in $EXTRA; do echo "== $v"; timeout 120 ./tc_probe_$v; done
  exit 0
fi
$NVCC $FL tc_probe.cu -o tc_probe_base &
$NVCC $FL -DKGQ_TC_TRACE tc_probe.cu -o tc_probe_trace &
$NVCC $FL tc_bn_check.cu -o tc_bn_check &
declare -A DEF=([nostore]="-DKGQ_TC_TRACE -DKGQ_TC_DBG_NO_STORE" [drain3]="-DKGQ_TC_TRACE -DKGQ_TC_DRAIN=3"
               [drain4]="-DKGQ_TC_TRACE -DKGQ_TC_DRAIN=4" [nobackoff]="-DKGQ_TC_NO_BACKOFF" [notma]="-DKGQ_TC_DBG_NO_TMA"
               [notma_nodrain]="-DKGQ_TC_DBG_NO_TMA -DKGQ_TC_DBG_NO_DRAIN" [notma_nostore]="-DKGQ_TC_DBG_NO_TMA -DKGQ_TC_DBG_NO_STORE"
               [notma_nodrain_nostore]="-DKGQ_TC_DBG_NO_TMA -DKGQ_TC_DBG_NO_DRAIN -DKGQ_TC_DBG_NO_STORE"
               [drain8]="-DKGQ_TC_DRAIN=8")
$NVCC $FL -DKGQ_TC_DRAIN=4 tc_bn_check.cu -o tc_bn_check_drain4 &
for v in $EXTRA; do $NVCC $FL ${DEF[$v]} tc_probe.cu -o tc_probe_$v & done
wait
ls tc_probe_* tc_bn_check
