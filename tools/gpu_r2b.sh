# round 2: re-run the changed / failing tests, GEMM split-K, small bench, XL launch list
cd $GRAFT_REPO_ROOT
export NNT_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_b.jsonl
rm -f $NNT_PARITY_LOG
timeout 1500 python -m pytest -q --timeout 900 -p no:cacheprovider -rf tests/test_gpu_block.py tests/test_gpu_kernels.py \
  tests/test_gpu_gemm.py tests/test_gpu_tp.py tests/test_gpu_dp_multirank.py tests/test_gpu_dp.py tests/test_gpu_gpt2.py \
  "tests/test_gpu_parity_full.py::test_gpt2_multistep_gradients_vs_oracle" > gpurun_out/pytest_b.log 2>&1
tail -15 gpurun_out/pytest_b.log
unset NNT_PARITY_LOG
timeout 600 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_b.log 2>&1; tail -c 400 gpurun_out/bench_small_b.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_xl2.csv python tools/profile_step.py --config xl --layers 2 > gpurun_out/ncu_xl2.log 2>&1
tail -2 gpurun_out/ncu_xl2.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_small.csv python tools/profile_step.py --config small > gpurun_out/ncu_small.log 2>&1
tail -2 gpurun_out/ncu_small.log
