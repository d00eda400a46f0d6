# LN forward groups / LN backward stats prefetch / embedding key sort: tests + micro-timings + XL step
cd $GRAFT_REPO_ROOT
timeout -s KILL 1200 python -m pytest -q --timeout 900 -p no:cacheprovider -rf tests/test_gpu_kernels.py tests/test_gpu_gpt2.py \
   tests/test_gpu_gemm.py tests/test_gpu_shapes.py > gpurun_out/pytest_r.log 2>&1
echo "tests rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_r.log | tail -12
for cfg in xl small; do
  for v in 0 1; do
    echo "== mem_bench $cfg NNT_LN_FWD_CTA=$v"
    NNT_LN_FWD_CTA=$v timeout -s KILL 300 python tools/mem_bench.py --config $cfg 2>&1 | tail -12
  done
done
for i in 1 2; do
  timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_r$i.log 2>&1
  python tools/summarize.py gpurun_out/bench_xl_r$i.log
done
