cd $GRAFT_REPO_ROOT
export NNT_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_j.jsonl
rm -f $NNT_PARITY_LOG
timeout -s KILL 2400 python -m pytest tests -m gpu -q --timeout 1800 -p no:cacheprovider -rf > gpurun_out/pytest_j.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_j.log
unset NNT_PARITY_LOG
timeout -s KILL 180 python __graft_entry__.py smoke > gpurun_out/smoke_j.log 2>&1; tail -1 gpurun_out/smoke_j.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_xl_j.log 2>&1; python tools/summarize.py gpurun_out/bench_xl_j.log
timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_j.log 2>&1; python tools/summarize.py gpurun_out/bench_small_j.log | head -4
bash tools/gpu_sanitize.sh > gpurun_out/sanitize_j.log 2>&1; cat gpurun_out/sanitize_j.log
