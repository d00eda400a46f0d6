# round-2 closing check at HEAD (after the 192-wide pair exception): full GPU suite, smoke, bench XL (default,
# with the CPU baseline) and small, small per-class traffic
cd $GRAFT_REPO_ROOT
timeout -s KILL 2400 python -m pytest tests -m gpu -q --timeout 1800 -p no:cacheprovider -rf > gpurun_out/pytest_final2.log 2>&1
echo "pytest rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_final2.log | tail -12
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke_final2.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final2.log
timeout -s KILL 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none --csv --log-file gpurun_out/traffic_small2.csv python tools/profile_step.py --config small --trace gpurun_out/trace_small2.json \
   > gpurun_out/ncu_traffic_small2.log 2>&1
python tools/traffic.py gpurun_out/traffic_small2.csv gpurun_out/trace_small2.json gpurun_out/traffic_small2.json | head -10
timeout -s KILL 900 python bench.py > gpurun_out/bench_xl_final2.log 2>&1; echo "bench default rc=$?"; python tools/summarize.py gpurun_out/bench_xl_final2.log
timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 > gpurun_out/bench_small_final2.log 2>&1; python tools/summarize.py gpurun_out/bench_small_final2.log | head -3
