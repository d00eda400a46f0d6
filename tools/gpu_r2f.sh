cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest -q --timeout 300 -p no:cacheprovider -rf tests/test_gpu_attention.py tests/test_gpu_tp.py \
   tests/test_gpu_block.py tests/test_gpu_gemm.py > gpurun_out/pytest_f.log 2>&1
echo "rc=$?"; grep -E "^E  |passed|failed" gpurun_out/pytest_f.log | head -20
for i in 1 2; do
timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_f.log 2>&1
python tools/summarize.py gpurun_out/bench_small_f.log | head -3
done
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_f.log 2>&1; python tools/summarize.py gpurun_out/bench_xl_f.log
NNT_GEMM_NO192=1 timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_f0.log 2>&1; python tools/summarize.py gpurun_out/bench_xl_f0.log | head -3
timeout -s KILL 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:attn_" -c 4 \
   -o gpurun_out/prof_attn2 -f python tools/profile_step.py --config small --layers 2 > gpurun_out/ncu_attn2.log 2>&1
tail -1 gpurun_out/ncu_attn2.log
timeout -s KILL 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_xl2_f.csv python tools/profile_step.py --config xl --layers 2 > gpurun_out/ncu_xl2_f.log 2>&1
python tools/summarize.py gpurun_out/launches_xl2_f.csv | head -14
