# narrow tail tiles v2 (MN-major granularity, tail-last only with K-major A) + ZeRO world-1 fix
cd $GRAFT_REPO_ROOT
timeout -s KILL 1500 python -m pytest -q --timeout 900 -p no:cacheprovider -rf tests/test_gpu_gemm.py \
  tests/test_gpu_dp.py tests/test_gpu_dp_multirank.py > gpurun_out/pytest_s3c.log 2>&1
echo "tests rc=$?"; grep -E "^(FAILED|ERROR)|^E  |passed|failed" gpurun_out/pytest_s3c.log | head -30
for t in 0 1 0 1; do
  NNT_GEMM_TAIL=$t timeout -s KILL 300 python tools/gemm_bench.py --config xl \
    --only out,proj,fc_dx,out_dx,qkv_dx,qkv_dw,fc_dw,out_dw,proj_dw > gpurun_out/gemm_tail$t.log 2>&1
  echo "== TAIL=$t"; cat gpurun_out/gemm_tail$t.log | tail -11
done
AB_ENV=NNT_GEMM_TAIL AB_N=3 bash tools/ab_env_bench.sh
