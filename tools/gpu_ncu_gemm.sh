cd $GRAFT_REPO_ROOT
for ONLY in $ONLYS; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 3 -c 1 -o gpurun_out/prof_gemm_$ONLY -f python tools/gemm_bench.py --only $ONLY --iters 1 > gpurun_out/ncu_gemm.log 2>&1
tail -1 gpurun_out/ncu_gemm.log
done
