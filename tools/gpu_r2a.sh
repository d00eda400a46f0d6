# round 2, first GPU pass: full GPU suite with the parity log, smoke, the default bench (XL)
cd $GRAFT_REPO_ROOT
export NNT_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity.jsonl
rm -f $NNT_PARITY_LOG
timeout 2400 python -m pytest tests -m gpu -q --timeout 1800 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1
tail -40 gpurun_out/pytest_gpu.log
unset NNT_PARITY_LOG
timeout 180 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_xl.log 2>&1; tail -c 1500 gpurun_out/bench_xl.log
