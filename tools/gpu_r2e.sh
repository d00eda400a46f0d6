cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python -m pytest -q --timeout 240 -p no:cacheprovider -rf tests/test_gpu_attention.py tests/test_gpu_tp.py \
   tests/test_gpu_gemm.py -k "attention or tp_stack or split_k" > gpurun_out/pytest_e.log 2>&1
echo "rc=$?"; grep -E "^E  |passed|failed" gpurun_out/pytest_e.log | head -20
timeout -s KILL 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:attn_" -c 2 \
   -o gpurun_out/prof_attn -f python tools/profile_step.py --config small --layers 2 > gpurun_out/ncu_attn.log 2>&1
tail -3 gpurun_out/ncu_attn.log
