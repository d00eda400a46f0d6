cd $GRAFT_REPO_ROOT
NNT_GEMM_MC=1 timeout 240 python -m pytest tests/test_gpu_gemm.py -q -x --timeout 120 -p no:cacheprovider 2>&1 | tail -15
for mc in 0 1; do
  echo "MC=$mc"
  NNT_GEMM_MC=$mc timeout 200 python tools/gemm_bench.py --only "qkv,fc+gelu,fc_plain,proj,proj_dx+gelu',fc_dx,qkv_dx,out_dx,proj_dw,fc_dw,square8192" 2>&1 | grep -v "^gemm\|total"
done
