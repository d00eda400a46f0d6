# round-2 session-3 re-entry check: full GPU suite, smoke, bench (default XL and small), XL one-step launch list
cd $GRAFT_REPO_ROOT
export NNT_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_s3a.jsonl
rm -f $NNT_PARITY_LOG
timeout -s KILL 2400 python -m pytest tests -m gpu -q --timeout 1800 -p no:cacheprovider -rf > gpurun_out/pytest_s3a.log 2>&1
echo "pytest rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_s3a.log | tail -25
unset NNT_PARITY_LOG
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke_s3a.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_s3a.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_xl_s3a.log 2>&1; echo "bench xl rc=$?"; python tools/summarize.py gpurun_out/bench_xl_s3a.log
timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_s3a.log 2>&1; python tools/summarize.py gpurun_out/bench_small_s3a.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_xl_s3a.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_xl_s3a.log 2>&1; echo "ncu rc=$?"
python tools/summarize.py gpurun_out/launches_xl_s3a.csv | head -40
