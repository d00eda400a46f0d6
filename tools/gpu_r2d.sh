cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python -m pytest -q -x --timeout 240 -p no:cacheprovider -rf tests/test_gpu_attention.py > gpurun_out/pytest_attn.log 2>&1
echo "attn rc=$?"; tail -30 gpurun_out/pytest_attn.log
timeout -s KILL 1500 python -m pytest -q --timeout 900 -p no:cacheprovider -rf tests/test_gpu_block.py tests/test_gpu_shapes.py \
   tests/test_gpu_gpt2.py tests/test_gpu_tp.py tests/test_gpu_parity_full.py tests/test_gpu_gemm.py > gpurun_out/pytest_d.log 2>&1
echo "rest rc=$?"; tail -12 gpurun_out/pytest_d.log
for env in "NNT_ATTN_FUSED=1" "NNT_ATTN_FUSED=0" ; do
  env $env timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_$env.log 2>&1
  echo $env; python tools/summarize.py gpurun_out/bench_small_$env.log | head -4
done
for env in "NNT_SPLITK_FUSED=0" "NNT_SPLITK_FUSED=1" "NNT_SPLITK_FUSED=0"; do
  env $env timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_sk.log 2>&1
  echo $env; python tools/summarize.py gpurun_out/bench_small_sk.log | head -2
done
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_d.log 2>&1; python tools/summarize.py gpurun_out/bench_xl_d.log
timeout -s KILL 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_small_d.csv python tools/profile_step.py --config small > gpurun_out/ncu_small_d.log 2>&1
python tools/summarize.py gpurun_out/launches_small_d.csv | head -20
