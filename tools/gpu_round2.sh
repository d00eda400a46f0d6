cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_dp.py tests/test_gpu_shapes.py -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_new.log 2>&1
tail -15 gpurun_out/pytest_new.log
timeout 300 python tools/gemm_bench.py > gpurun_out/gemm_bench.log 2>&1; cat gpurun_out/gemm_bench.log
ONLYS="fc+gelu out proj pv" bash tools/gpu_ncu_gemm.sh
ls gpurun_out
