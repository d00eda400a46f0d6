# dedicated attention row-statistics kernel: tests, kernel times, step A/B
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest -q --timeout 600 -p no:cacheprovider -rf tests/test_gpu_attention.py tests/test_gpu_block.py \
   tests/test_gpu_parity_full.py > gpurun_out/pytest_aa.log 2>&1
echo "tests rc=$?"; grep -E "^(FAILED|ERROR)|^E  |passed|failed" gpurun_out/pytest_aa.log | head -20
for v in 1 0; do
  NNT_ATTN_STATS=$v timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --kernel-name-base demangled -k "regex:attn_stats|gemm_tc_kernel<\(int\)128, float, \(int\)3" -c 3 --log-file gpurun_out/stats$v.csv \
    python tools/profile_step.py --config xl > /dev/null 2>&1
  echo "stats=$v"; grep gpu__time gpurun_out/stats$v.csv | awk -F'","' '{print substr($5,1,50)" "$NF}'
done
for r in 1 2; do for v in 1 0; do
  NNT_ATTN_STATS=$v timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_aa$v$r.log 2>&1
  echo "xl stats=$v"; python tools/summarize.py gpurun_out/bench_xl_aa$v$r.log | head -3
done; done
for v in 1 0; do
  NNT_ATTN_STATS=$v timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_aa$v.log 2>&1
  echo "small stats=$v"; python tools/summarize.py gpurun_out/bench_small_aa$v.log | head -3
done
