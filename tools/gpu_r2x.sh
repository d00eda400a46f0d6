# attention L2 policy modes 0 / 1 / 2, interleaved XL steps; backward kernel DRAM bytes per mode
cd $GRAFT_REPO_ROOT
for v in 0 1 2; do
  NNT_ATTN_L2HINT=$v timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --kernel-name-base demangled -k "regex:attn_bwd" -c 2 --log-file gpurun_out/attn_bwd_hint$v.csv \
    python tools/profile_step.py --config xl > /dev/null 2>&1
done
for r in 1 2; do for v in 2 0 1; do
  NNT_ATTN_L2HINT=$v timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_x$v$r.log 2>&1
  echo "xl hint=$v"; python tools/summarize.py gpurun_out/bench_xl_x$v$r.log | head -3
done; done
