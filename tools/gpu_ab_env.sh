# A/B of an env switch: parity tests with the default, then mem_bench + bench with and without $AB_ENV=1
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_block.py tests/test_gpu_gpt2.py -q --timeout 200 -p no:cacheprovider 2>&1 | tail -2
for v in 0 1; do
  echo "== $AB_ENV=$v"
  env $AB_ENV=$v timeout 200 python tools/mem_bench.py 2>&1 | grep -E "kernel|${AB_GREP:-.}"
  env $AB_ENV=$v timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_ab$v.log 2>&1; python tools/summarize.py gpurun_out/bench_ab$v.log | head -4
done
