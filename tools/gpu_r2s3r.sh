# fp32 residual TMA-staged through the epilogue staging ring (NNT_GEMM_RES_SMEM): tests, GEMM micro A/B, step A/B
cd $GRAFT_REPO_ROOT
timeout -s KILL 1500 python -m pytest -q --timeout 900 -p no:cacheprovider -rf tests/test_gpu_gemm.py \
  tests/test_gpu_block.py tests/test_gpu_shapes.py tests/test_gpu_parity_full.py > gpurun_out/pytest_s3r.log 2>&1
echo "tests rc=$?"; grep -E "^(FAILED|ERROR)|^E  |passed|failed" gpurun_out/pytest_s3r.log | head -20
for v in 0 1 0 1; do
  NNT_GEMM_RES_SMEM=$v timeout -s KILL 300 python tools/gemm_bench.py --config xl --only out,proj > gpurun_out/rs$v.log 2>&1
  echo "== XL RES_SMEM=$v"; tail -3 gpurun_out/rs$v.log
  NNT_GEMM_RES_SMEM=$v timeout -s KILL 300 python tools/gemm_bench.py --config small --only out,proj > gpurun_out/rss$v.log 2>&1
  echo "== small RES_SMEM=$v"; tail -3 gpurun_out/rss$v.log
done
AB_ENV=NNT_GEMM_RES_SMEM AB_N=3 bash tools/ab_env_bench.sh
AB_ENV=NNT_GEMM_RES_SMEM AB_N=3 BENCH_ARGS="--config small" bash tools/ab_env_bench.sh
