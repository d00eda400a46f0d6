cd $GRAFT_REPO_ROOT
free -g | head -2
timeout -s KILL 300 python tools/attn_trace.py --config small > gpurun_out/attn_trace.txt 2>&1; head -60 gpurun_out/attn_trace.txt
timeout -s KILL 600 python -m pytest -q --timeout 300 -p no:cacheprovider -rf tests/test_gpu_offload.py > gpurun_out/pytest_h.log 2>&1
echo "rc=$?"; grep -E "^E  |passed|failed" gpurun_out/pytest_h.log | head -10
