cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_gemm.py tests/test_gpu_block.py tests/test_gpu_gpt2.py tests/test_gpu_dp.py tests/test_gpu_loss_reader.py -q --timeout 300 -p no:cacheprovider 2>&1 | tail -2
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_sk.csv python tools/profile_step.py > /dev/null 2>&1
python tools/summarize.py gpurun_out/launches_sk.csv | grep -E "launches|splitk|colsum"
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sk.log 2>&1; python tools/summarize.py gpurun_out/bench_sk.log | head -2
