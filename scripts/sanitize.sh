#!/bin/bash
# compute-sanitizer over the library on small configs: memcheck (out-of-bounds /
# misaligned accesses, leaks), racecheck (shared-memory hazards), synccheck (barrier misuse) on
#   * the BetaE path with split-K GEMM tails (d 128, H 512, 300 queries: publish / last-arriver
#     reduce with acq_rel fences), the tensor-core scorer and block-minima top-k,
#   * the N2 peer push / merge protocol (three virtual ranks),
#   * GQE / Q2B SIMT scorers (tiled and TMA-streamed) and the filtered rank.
# Each tool runs scripts/sanitize_case.py under `compute-sanitizer --tool T`; the summaries are
# the evidence (profiles/r02/sanitize_*.txt).
cd "$(dirname "$0")/.."
for tool in memcheck racecheck synccheck; do
  echo "=== $tool"
  KGQ_NO_GRAPHS=1 timeout 1500 compute-sanitizer --tool $tool --print-limit 200 python scripts/sanitize_case.py \
    > gpurun_out/sanitize_$tool.log 2>&1
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|^case|all cases" gpurun_out/sanitize_$tool.log
done
# the tcgen05 GEMM alone (every tile width, epilogue form and split-K tail) under racecheck
( cd scripts && [ -x tc_bn_check ] && timeout 900 compute-sanitizer --tool racecheck --print-limit 200 ./tc_bn_check ) \
  > gpurun_out/sanitize_racecheck_gemm.log 2>&1
grep -E "RACECHECK SUMMARY|all tile widths|FAILED" gpurun_out/sanitize_racecheck_gemm.log
