# attention TMA L2 cache policies: tests, interleaved XL / small A/B, per-kernel ncu list; rowstats --set full
cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest -q --timeout 500 -p no:cacheprovider -rf tests/test_gpu_attention.py tests/test_gpu_block.py > gpurun_out/pytest_w.log 2>&1
echo "tests rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_w.log | tail -5
for v in 1 0; do
  NNT_ATTN_L2HINT=$v timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --kernel-name-base demangled -k "regex:attn_" -c 4 --log-file gpurun_out/attn_hint$v.csv \
    python tools/profile_step.py --config xl > /dev/null 2>&1
  echo "hint=$v"; grep -E "gpu__time|dram__bytes" gpurun_out/attn_hint$v.csv | awk -F'","' '{print $5" "$(NF-2)" "$NF}' | cut -c1-120 | head -12
done
for v in 1 0 1 0; do
  NNT_ATTN_L2HINT=$v timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_w$v.log 2>&1
  echo "xl hint=$v"; python tools/summarize.py gpurun_out/bench_xl_w$v.log | head -3
done
for v in 1 0; do
  NNT_ATTN_L2HINT=$v timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_w$v.log 2>&1
  echo "small hint=$v"; python tools/summarize.py gpurun_out/bench_small_w$v.log | head -3
done
timeout -s KILL 600 ncu --profile-from-start off --set full --import-source on --clock-control none \
   --kernel-name-base demangled -k "regex:gemm_tc_kernel<\(int\)128, float, \(int\)3" -s 2 -c 1 -o gpurun_out/prof_w_rowstats -f \
   python tools/profile_step.py --config xl > gpurun_out/ncu_w_rowstats.log 2>&1; tail -1 gpurun_out/ncu_w_rowstats.log
