# out-projection (8192x1600x1600, fp32 residual) tile choice: single-CTA 192 (default) vs 256-wide pairs with the narrow tail
cd $GRAFT_REPO_ROOT
for i in 1 2; do
NNT_DEBUG_GEMM=1 timeout -s KILL 300 python tools/gemm_bench.py --config xl --only out,out_dx,proj > gpurun_out/o_def.log 2>gpurun_out/o_def.err
echo "== default"; tail -4 gpurun_out/o_def.log; grep launch gpurun_out/o_def.err | sort | uniq -c
NNT_GEMM_CG=2 NNT_GEMM_BN=256 NNT_DEBUG_GEMM=1 timeout -s KILL 300 python tools/gemm_bench.py --config xl --only out,out_dx,proj > gpurun_out/o_p256.log 2>gpurun_out/o_p256.err
echo "== pair 256"; tail -4 gpurun_out/o_p256.log; grep launch gpurun_out/o_p256.err | sort | uniq -c
done
