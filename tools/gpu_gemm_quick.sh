# quick GEMM timing + GEMM parity tests
cd $GRAFT_REPO_ROOT
timeout 300 python tools/gemm_bench.py --only ${ONLY:-qkv,out,fc+gelu,proj,proj_dx+gelu\',fc_dx,out_dx,qkv_dx,proj_dw,fc_dw,out_dw,qkv_dw} 2>&1 | tail -14
if [ -n "$TESTS" ]; then timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -3; fi
