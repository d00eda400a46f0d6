# GPU round trip: parity tests, smoke, bench, one-step ncu launch list (+ optional full capture)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 180 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -15 gpurun_out/pytest_gpu.log
timeout 180 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; tail -c 600 gpurun_out/bench.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv python tools/profile_step.py > gpurun_out/ncu_list.log 2>&1
tail -3 gpurun_out/ncu_list.log
timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/profile_step.py --trace gpurun_out/trace.json \
   > gpurun_out/ncu_traffic.log 2>&1
python tools/traffic.py gpurun_out/traffic.csv gpurun_out/trace.json gpurun_out/traffic_small.json
if [ -n "$NCU_FULL" ]; then
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
     -k "regex:$NCU_FULL" -c ${NCU_COUNT:-4} -o gpurun_out/prof_full -f python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
  tail -3 gpurun_out/ncu_full.log
fi
