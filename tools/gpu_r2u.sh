# attention backward with dA formed in place (3 stages), LN backward rings: tests, timings; focused sanitizer logs
cd $GRAFT_REPO_ROOT
timeout -s KILL 1500 python -m pytest -q --timeout 900 -p no:cacheprovider -rf tests/test_gpu_attention.py tests/test_gpu_kernels.py \
   tests/test_gpu_block.py tests/test_gpu_parity_full.py tests/test_gpu_shapes.py > gpurun_out/pytest_u.log 2>&1
echo "tests rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_u.log | tail -12
timeout -s KILL 300 python tools/attn_trace.py --config small > gpurun_out/attn_trace_u.txt 2>&1; tail -25 gpurun_out/attn_trace_u.txt
timeout -s KILL 300 python tools/mem_bench.py --config xl --only ln_bwd 2>&1 | tail -3
NNT_LN_BWD_RING=0 timeout -s KILL 300 python tools/mem_bench.py --config xl --only ln_bwd 2>&1 | tail -2
timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_u.log 2>&1; python tools/summarize.py gpurun_out/bench_small_u.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_u.log 2>&1; python tools/summarize.py gpurun_out/bench_xl_u.log
timeout -s KILL 600 compute-sanitizer --tool racecheck --print-limit 40 python -m pytest -q -p no:cacheprovider --timeout 500 \
  "tests/test_gpu_gemm.py::test_gemm_cta_pair_bit_exact" > gpurun_out/racecheck_u.log 2>&1; grep -v "^\.\+" gpurun_out/racecheck_u.log | head -60
timeout -s KILL 900 compute-sanitizer --tool initcheck --print-limit 30 python -m pytest -q -p no:cacheprovider --timeout 800 \
  "tests/test_gpu_dp.py::test_dp_path_world1_equals_single_gpu_bitwise" > gpurun_out/initcheck_u.log 2>&1; grep -E "Uninitialized|at |in |ERROR SUMMARY|FAILED|passed|failed" gpurun_out/initcheck_u.log | head -60
