cd $GRAFT_REPO_ROOT
export NNT_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_c.jsonl
rm -f $NNT_PARITY_LOG
timeout 2400 python -m pytest -q --timeout 1800 -p no:cacheprovider -rf tests -m gpu > gpurun_out/pytest_c.log 2>&1
tail -12 gpurun_out/pytest_c.log
unset NNT_PARITY_LOG
timeout 600 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_c.log 2>&1; tail -c 300 gpurun_out/bench_small_c.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_c.log 2>&1; tail -c 300 gpurun_out/bench_xl_c.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_small_c.csv python tools/profile_step.py --config small > gpurun_out/ncu_small_c.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_xl2_c.csv python tools/profile_step.py --config xl --layers 2 > gpurun_out/ncu_xl2_c.log 2>&1
