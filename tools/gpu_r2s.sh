# ncu --set full of XL projection GEMMs: K-major proj_plain vs MN-major-B fc_dx vs MN-major-both dW
cd $GRAFT_REPO_ROOT
for ONLY in ${ONLYS:-proj_plain fc_dx fc_dw}; do
  timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 3 -c 1 \
     -o gpurun_out/prof_g_$ONLY -f python tools/gemm_bench.py --config xl --only $ONLY --iters 1 --no-ws > gpurun_out/ncu_g_$ONLY.log 2>&1
  tail -1 gpurun_out/ncu_g_$ONLY.log
done
