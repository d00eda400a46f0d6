cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest -q --timeout 300 -p no:cacheprovider -rf tests/test_gpu_attention.py tests/test_gpu_tp.py \
   tests/test_gpu_block.py tests/test_gpu_offload.py > gpurun_out/pytest_g.log 2>&1
echo "rc=$?"; grep -E "^E  |passed|failed" gpurun_out/pytest_g.log | head -20
timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_g.log 2>&1
python tools/summarize.py gpurun_out/bench_small_g.log | head -3
timeout -s KILL 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:attn_" -c 4 \
   -o gpurun_out/prof_attn3 -f python tools/profile_step.py --config small --layers 2 > gpurun_out/ncu_attn3.log 2>&1
tail -1 gpurun_out/ncu_attn3.log
