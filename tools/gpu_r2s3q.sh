# split K in two for the short-grid fp32 dX GEMMs (NNT_GEMM_SPLIT2): tests + small step A/B + XL check
cd $GRAFT_REPO_ROOT
NNT_DEBUG_GEMM=1 timeout -s KILL 300 python tools/gemm_bench.py --config small --only fc_dx,qkv_dx,out_dx 2>gpurun_out/s2.err | tail -4
grep launch gpurun_out/s2.err | sort | uniq -c
NNT_GEMM_SPLIT2=0 timeout -s KILL 300 python tools/gemm_bench.py --config small --only fc_dx,qkv_dx,out_dx | tail -4
timeout -s KILL 1500 python -m pytest -q --timeout 900 -p no:cacheprovider -rf tests/test_gpu_gemm.py \
  tests/test_gpu_block.py tests/test_gpu_parity_full.py tests/test_gpu_shapes.py tests/test_gpu_dp.py > gpurun_out/pytest_s3q.log 2>&1
echo "tests rc=$?"; grep -E "^(FAILED|ERROR)|^E  |passed|failed" gpurun_out/pytest_s3q.log | head -20
AB_ENV=NNT_GEMM_SPLIT2 AB_N=4 BENCH_ARGS="--config small" bash tools/ab_env_bench.sh
AB_ENV=NNT_GEMM_SPLIT2 AB_N=1 bash tools/ab_env_bench.sh
