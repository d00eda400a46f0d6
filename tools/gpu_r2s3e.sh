# stream-K re-check on top of the blocked MN-major maps and narrow tails
cd $GRAFT_REPO_ROOT
for v in 0 1; do
  NNT_GEMM_SK=$v NNT_DEBUG_GEMM=1 timeout -s KILL 300 python tools/gemm_bench.py --config xl \
    --only proj,fc_dx,qkv_dx,qkv_dw,fc_dw,out_dw,proj_dw > gpurun_out/gemm_sk$v.log 2>gpurun_out/gemm_sk$v.err
  echo "== SK=$v"; cat gpurun_out/gemm_sk$v.log | tail -9; grep -c stream-K gpurun_out/gemm_sk$v.err
done
AB_ENV=NNT_GEMM_SK AB_N=3 bash tools/ab_env_bench.sh
