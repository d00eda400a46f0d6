# round-2 final validation: full GPU suite (+ parity log), smoke, per-class DRAM traffic (xl, small: the bench's
# roofline "traffic" source), bench XL (default) / small / large / wide / reference arm, XL one-step launch list,
# ncu --set full of the dominant GEMM class in the XL step
cd $GRAFT_REPO_ROOT
export NNT_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_final.jsonl
rm -f $NNT_PARITY_LOG
timeout -s KILL 2400 python -m pytest tests -m gpu -q --timeout 1800 -p no:cacheprovider -rf > gpurun_out/pytest_final.log 2>&1
echo "pytest rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_final.log | tail -12
unset NNT_PARITY_LOG
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final.log
for cfg in xl small; do
timeout -s KILL 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none --csv --log-file gpurun_out/traffic_$cfg.csv python tools/profile_step.py --config $cfg --trace gpurun_out/trace_$cfg.json \
   > gpurun_out/ncu_traffic_$cfg.log 2>&1
python tools/traffic.py gpurun_out/traffic_$cfg.csv gpurun_out/trace_$cfg.json gpurun_out/traffic_$cfg.json | head -12
done
timeout -s KILL 900 python bench.py > gpurun_out/bench_xl_final.log 2>&1; echo "bench default rc=$?"; python tools/summarize.py gpurun_out/bench_xl_final.log
timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 > gpurun_out/bench_small_final.log 2>&1; python tools/summarize.py gpurun_out/bench_small_final.log | head -3
timeout -s KILL 600 python bench.py --config large --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_large_final.log 2>&1; python tools/summarize.py gpurun_out/bench_large_final.log | head -3
timeout -s KILL 600 python bench.py --config wide --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_wide_final.log 2>&1; python tools/summarize.py gpurun_out/bench_wide_final.log | head -3
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_final.log 2>&1; tail -c 400 gpurun_out/bench_ref_final.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_xl_final.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_xl_final.log 2>&1; echo "ncu list rc=$?"
python tools/summarize.py gpurun_out/launches_xl_final.csv | head -30
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 40 -c 1 \
  -o gpurun_out/prof_final_gemm -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full_final.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py gpurun_out/prof_final_gemm.ncu-rep | tee gpurun_out/ncu_full_final_summary.txt
ls -la gpurun_out/prof_final_gemm.ncu-rep
