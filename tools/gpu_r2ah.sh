# split-major split-K task order: GEMM tests, LM-head dh GEMM DRAM bytes / time, step A/B
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest -q --timeout 600 -p no:cacheprovider -rf tests/test_gpu_gemm.py tests/test_gpu_gpt2.py > gpurun_out/pytest_ah.log 2>&1
echo "tests rc=$?"; grep -E "^(FAILED|ERROR)|^E  |passed|failed" gpurun_out/pytest_ah.log | head -10
for v in 1 0; do
  NNT_GEMM_SPLITMAJOR=$v timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --kernel-name-base demangled -k "regex:gemm_tc_kernel<\(int\)256, float" -s 97 -c 2 --log-file gpurun_out/sm$v.csv \
    python tools/profile_step.py --config xl > /dev/null 2>&1
  echo "splitmajor=$v"; grep -E "gpu__time|dram__bytes" gpurun_out/sm$v.csv | awk -F'","' '{print $(NF-2)" "$NF}'
done
for r in 1 2; do for v in 1 0; do
  NNT_GEMM_SPLITMAJOR=$v timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_ah$v$r.log 2>&1
  echo "xl splitmajor=$v"; python tools/summarize.py gpurun_out/bench_xl_ah$v$r.log | head -2
done; done
