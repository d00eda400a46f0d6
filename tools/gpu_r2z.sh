# R35 fused tensor-parallel SUM: TP tests (ranks standing in one process, world-1 stack), GEMM / block regression
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest -q --timeout 600 -p no:cacheprovider -rf tests/test_gpu_tp.py tests/test_gpu_gemm.py \
   tests/test_gpu_block.py > gpurun_out/pytest_z.log 2>&1
echo "tests rc=$?"; grep -E "^(FAILED|ERROR)|^E  |passed|failed" gpurun_out/pytest_z.log | head -30
timeout -s KILL 300 python tools/tp_bench.py --help > /dev/null 2>&1; echo "tp_bench present rc=$?"
