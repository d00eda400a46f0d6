cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python tools/attn_trace.py --config small > gpurun_out/attn_trace.txt 2>&1; head -40 gpurun_out/attn_trace.txt
timeout -s KILL 600 python -m pytest -q --timeout 300 -p no:cacheprovider -rf tests/test_gpu_attention.py tests/test_gpu_block.py -k "attention or bf16" > gpurun_out/pytest_i.log 2>&1
echo "rc=$?"; grep -E "^E  |passed|failed" gpurun_out/pytest_i.log | head -10
timeout -s KILL 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_small_i.csv python tools/profile_step.py --config small --layers 2 > /dev/null 2>&1
python tools/summarize.py gpurun_out/launches_small_i.csv | grep attn
