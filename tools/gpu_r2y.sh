# round-2 validation: full GPU suite (+ parity log), smoke, bench XL (default) / small / large / wide,
# one-step XL launch list + per-class DRAM traffic (the bench's roofline "traffic" source)
cd $GRAFT_REPO_ROOT
export NNT_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_y.jsonl
rm -f $NNT_PARITY_LOG
timeout -s KILL 2400 python -m pytest tests -m gpu -q --timeout 1800 -p no:cacheprovider -rf > gpurun_out/pytest_y.log 2>&1
echo "pytest rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_y.log | tail -12
unset NNT_PARITY_LOG
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke_y.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_y.log
timeout -s KILL 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none --csv --log-file gpurun_out/traffic_xl_y.csv python tools/profile_step.py --config xl --trace gpurun_out/trace_xl_y.json \
   > gpurun_out/ncu_traffic_xl_y.log 2>&1
python tools/traffic.py gpurun_out/traffic_xl_y.csv gpurun_out/trace_xl_y.json gpurun_out/traffic_xl_y.json | head -10
timeout -s KILL 900 python bench.py > gpurun_out/bench_xl_y.log 2>&1; echo "bench default rc=$?"; python tools/summarize.py gpurun_out/bench_xl_y.log
timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 > gpurun_out/bench_small_y.log 2>&1; python tools/summarize.py gpurun_out/bench_small_y.log | head -3
timeout -s KILL 600 python bench.py --config large --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_large_y.log 2>&1; python tools/summarize.py gpurun_out/bench_large_y.log | head -3
timeout -s KILL 600 python bench.py --config wide --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_wide_y.log 2>&1; python tools/summarize.py gpurun_out/bench_wide_y.log | head -3
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_y.log 2>&1; tail -c 300 gpurun_out/bench_ref_y.log
