# ncu --set full of the XL attention kernels (rowstats GEMM epilogue, fused forward, new fused backward, dQ GEMM)
cd $GRAFT_REPO_ROOT
for K in "gemm_tc_kernel<128, float, 3" attn_fwd_pv_kernel attn_bwd_kv_kernel "gemm_tc_kernel<64, __nv_bfloat16"; do
  tag=$(echo "$K" | tr -cd 'a-z_0-9')
  timeout -s KILL 600 ncu --profile-from-start off --set full --import-source on --clock-control none \
     --kernel-name-base demangled -k "regex:$K" -s 2 -c 1 -o gpurun_out/prof_v_$tag -f \
     python tools/profile_step.py --config xl > gpurun_out/ncu_v_$tag.log 2>&1
  tail -1 gpurun_out/ncu_v_$tag.log
done
