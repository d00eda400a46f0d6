# 192-wide pair exception (K-major B, 256-wide pair rounds < 70 % full): tests + small step A/B + XL check
cd $GRAFT_REPO_ROOT
timeout -s KILL 1200 python -m pytest -q --timeout 900 -p no:cacheprovider -rf tests/test_gpu_gemm.py \
  tests/test_gpu_block.py tests/test_gpu_parity_full.py > gpurun_out/pytest_s3p.log 2>&1
echo "tests rc=$?"; grep -E "^(FAILED|ERROR)|^E  |passed|failed" gpurun_out/pytest_s3p.log | head -20
AB_ENV=NNT_GEMM_192_EXC AB_N=4 BENCH_ARGS="--config small" bash tools/ab_env_bench.sh
AB_ENV=NNT_GEMM_192_EXC AB_N=2 bash tools/ab_env_bench.sh
