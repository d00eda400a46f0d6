# stream-K / tile-choice sweep on the XL and small projection GEMMs, with the library's launch choices
cd $GRAFT_REPO_ROOT
G="qkv,out,fc+gelu,proj_plain,proj,proj_dw,proj_dx+gelu',fc_dw,fc_dx,out_dw,out_dx,qkv_dw,qkv_dx"
for cfg in xl small; do
for mode in "NNT_GEMM_SK=0" "NNT_GEMM_SK=1" "NNT_GEMM_SK=1 NNT_GEMM_BN=256" "NNT_GEMM_SK=0 NNT_GEMM_BN=256"; do
  echo "== $cfg $mode"
  env $mode NNT_DEBUG_GEMM=1 timeout -s KILL 300 python tools/gemm_bench.py --config $cfg --iters 8 --only "$G" > gpurun_out/gb.txt 2> gpurun_out/gb.err
  env $mode timeout -s KILL 300 python tools/gemm_bench.py --config $cfg --iters 20 --only "$G" > gpurun_out/gb.txt 2>&1
  sort -u gpurun_out/gb.err | grep launch | sed 's/gemm_tc launch //'
  cat gpurun_out/gb.txt
done
done
