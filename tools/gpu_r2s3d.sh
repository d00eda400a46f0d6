# blocked 5-D TMA maps for MN-major operands (NNT_GEMM_BLOCKED) on top of the narrow tails
cd $GRAFT_REPO_ROOT
timeout -s KILL 1500 python -m pytest -q --timeout 900 -p no:cacheprovider -rf tests/test_gpu_gemm.py \
  tests/test_gpu_block.py tests/test_gpu_shapes.py > gpurun_out/pytest_s3d.log 2>&1
echo "tests rc=$?"; grep -E "^(FAILED|ERROR)|^E  |passed|failed" gpurun_out/pytest_s3d.log | head -30
for t in 0 1 0 1; do
  NNT_GEMM_BLOCKED=$t timeout -s KILL 300 python tools/gemm_bench.py --config xl \
    --only proj_dx_plain,fc_dx,out_dx,qkv_dx,qkv_dw,fc_dw,out_dw,proj_dw,proj_dx+gelu\' > gpurun_out/gemm_blk$t.log 2>&1
  echo "== BLOCKED=$t"; cat gpurun_out/gemm_blk$t.log | tail -11
done
NNT_GEMM_BLOCKED=1 timeout -s KILL 300 python tools/gemm_bench.py --config small > gpurun_out/gemm_small_blk1.log 2>&1
NNT_GEMM_BLOCKED=0 timeout -s KILL 300 python tools/gemm_bench.py --config small > gpurun_out/gemm_small_blk0.log 2>&1
paste <(awk '{print $1, $(NF-1)}' gpurun_out/gemm_small_blk0.log) <(awk '{print $(NF-1)}' gpurun_out/gemm_small_blk1.log) | head -40
AB_ENV=NNT_GEMM_BLOCKED AB_N=3 bash tools/ab_env_bench.sh
AB_ENV=NNT_GEMM_BLOCKED AB_N=2 BENCH_ARGS="--config small" bash tools/ab_env_bench.sh
