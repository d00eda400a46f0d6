# ncu --set full of three XL GEMMs on the current path (fc_dx: K-major A / blocked MN-major B, fp32 out;
# proj_dw: both operands blocked MN-major; out: K = 1600 with the fp32 residual epilogue)
cd $GRAFT_REPO_ROOT
for ONLY in fc_dx proj_dw out proj; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 3 -c 1 \
  -o gpurun_out/prof_xl_$ONLY -f python tools/gemm_bench.py --config xl --only $ONLY --iters 1 > gpurun_out/ncu_gemm_$ONLY.log 2>&1
echo "$ONLY rc=$?"
done
python tools/ncu_summary.py gpurun_out/prof_xl_*.ncu-rep
