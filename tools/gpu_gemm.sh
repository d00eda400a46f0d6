cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_block.py -q --timeout 180 -p no:cacheprovider 2>&1 | tail -4
timeout 300 python tools/gemm_bench.py 2>&1 | tail -25
