# round-2 closing check at HEAD (TMA-staged residual, out-projection pair-256 rule): out GEMM micro check,
# full GPU suite, smoke, per-class traffic (xl, small), bench XL (default) / small / large / wide, XL launch list
cd $GRAFT_REPO_ROOT
NNT_DEBUG_GEMM=1 timeout -s KILL 300 python tools/gemm_bench.py --config xl --only out,proj 2>gpurun_out/o.err | tail -3; grep launch gpurun_out/o.err | sort | uniq -c
timeout -s KILL 300 python tools/gemm_bench.py --config small --only out,proj | tail -3
timeout -s KILL 2400 python -m pytest tests -m gpu -q --timeout 1800 -p no:cacheprovider -rf > gpurun_out/pytest_final3.log 2>&1
echo "pytest rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_final3.log | tail -12
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke_final3.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final3.log
for cfg in xl small; do
timeout -s KILL 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none --csv --log-file gpurun_out/traffic3_$cfg.csv python tools/profile_step.py --config $cfg --trace gpurun_out/trace3_$cfg.json \
   > gpurun_out/ncu_traffic3_$cfg.log 2>&1
python tools/traffic.py gpurun_out/traffic3_$cfg.csv gpurun_out/trace3_$cfg.json gpurun_out/traffic3_$cfg.json | head -3
done
timeout -s KILL 900 python bench.py > gpurun_out/bench_xl_final3.log 2>&1; echo "bench default rc=$?"; python tools/summarize.py gpurun_out/bench_xl_final3.log
timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 > gpurun_out/bench_small_final3.log 2>&1; python tools/summarize.py gpurun_out/bench_small_final3.log | head -3
timeout -s KILL 600 python bench.py --config large --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_large_final3.log 2>&1; python tools/summarize.py gpurun_out/bench_large_final3.log | head -2
timeout -s KILL 600 python bench.py --config wide --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_wide_final3.log 2>&1; python tools/summarize.py gpurun_out/bench_wide_final3.log | head -2
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_xl_final3.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_xl_final3.log 2>&1; echo "ncu list rc=$?"
python tools/summarize.py gpurun_out/launches_xl_final3.csv | head -16
