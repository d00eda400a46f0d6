# XL GEMM tile choice with narrow tails: default vs forced CTA pairs (NNT_GEMM_CG=2)
cd $GRAFT_REPO_ROOT
for cg in 0 2 0 2; do
  NNT_GEMM_CG=$cg NNT_DEBUG_GEMM=1 timeout -s KILL 300 python tools/gemm_bench.py --config xl \
    --only qkv,out,fc+gelu,proj,proj_dx+gelu\',fc_dx,out_dx,qkv_dx,qkv_dw,fc_dw,out_dw,proj_dw > gpurun_out/gemm_cg$cg.log 2>gpurun_out/gemm_cg$cg.err
  echo "== CG=$cg"; tail -14 gpurun_out/gemm_cg$cg.log; grep 'launch' gpurun_out/gemm_cg$cg.err | sort | uniq -c | head -14
done
