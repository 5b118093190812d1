cd $GRAFT_REPO_ROOT
bash scripts/tc_probe.sh run > gpurun_out/tc_probe.txt 2>&1
cat gpurun_out/tc_probe.txt
cd scripts
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 92 -c 1 -o ../gpurun_out/prof_score_probe ./tc_probe_base > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 23 -c 1 -o ../gpurun_out/prof_mlp_probe ./tc_probe_base > /dev/null 2>&1
ls ../gpurun_out
