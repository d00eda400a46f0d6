cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest -q --timeout 600 -p no:cacheprovider -rf tests/test_gpu_dp.py tests/test_gpu_offload.py \
   tests/test_gpu_gpt2.py tests/test_gpu_block.py tests/test_gpu_dp_multirank.py > gpurun_out/pytest_k.log 2>&1
echo "pytest rc=$?"; grep -E "^E  |passed|failed" gpurun_out/pytest_k.log | head
timeout -s KILL 300 python tools/attn_trace.py --config small > gpurun_out/attn_trace_bwd.txt 2>&1; sed -n '/backward/,$p' gpurun_out/attn_trace_bwd.txt | head -30
for v in 1 0 1 0; do
  NNT_OVERLAP_UPDATE=$v timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_k$v.log 2>&1
  echo "overlap=$v"; python tools/summarize.py gpurun_out/bench_small_k$v.log | head -1
done
for v in 1 0; do
  NNT_OVERLAP_UPDATE=$v timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_k$v.log 2>&1
  echo "xl overlap=$v"; python tools/summarize.py gpurun_out/bench_xl_k$v.log | head -1
done
timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --act-offload 48 --offload --no-cpu-baseline > gpurun_out/bench_xl_offload.log 2>&1
echo "xl act+opt offload"; python tools/summarize.py gpurun_out/bench_xl_offload.log | head -1
