# lagged side-stream join: bitwise tests, model / DP / offload regressions, interleaved XL / small A/B
cd $GRAFT_REPO_ROOT
timeout -s KILL 1200 python -m pytest -q --timeout 900 -p no:cacheprovider -rf tests/test_gpu_block.py tests/test_gpu_dp.py \
   tests/test_gpu_offload.py tests/test_gpu_gpt2.py tests/test_gpu_dp_multirank.py tests/test_gpu_parity_full.py > gpurun_out/pytest_ad.log 2>&1
echo "tests rc=$?"; grep -E "^(FAILED|ERROR)|^E  |passed|failed" gpurun_out/pytest_ad.log | head -20
for r in 1 2; do for v in 1 0; do
  NNT_SIDE_LAG=$v timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_ad$v$r.log 2>&1
  echo "xl lag=$v"; python tools/summarize.py gpurun_out/bench_xl_ad$v$r.log | head -1
  NNT_SIDE_LAG=$v timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_ad$v$r.log 2>&1
  echo "small lag=$v"; python tools/summarize.py gpurun_out/bench_small_ad$v$r.log | head -1
done; done
