# last check at HEAD: full GPU suite, smoke, default bench
cd $GRAFT_REPO_ROOT
timeout -s KILL 2400 python -m pytest tests -m gpu -q --timeout 1800 -p no:cacheprovider -rf > gpurun_out/pytest_final4.log 2>&1
echo "pytest rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_final4.log | tail -12
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke_final4.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final4.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_xl_final4.log 2>&1; echo "bench default rc=$?"; python tools/summarize.py gpurun_out/bench_xl_final4.log | head -4
