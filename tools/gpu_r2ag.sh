# per-kernel DRAM bytes of one XL step with the M-outer raster (ncu list with dram metrics)
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none --csv --log-file gpurun_out/traffic_xl_ag.csv python tools/profile_step.py --config xl --trace gpurun_out/trace_xl_ag.json \
   > gpurun_out/ncu_traffic_xl_ag.log 2>&1
python tools/traffic.py gpurun_out/traffic_xl_ag.csv gpurun_out/trace_xl_ag.json gpurun_out/traffic_xl_ag.json | head -10
