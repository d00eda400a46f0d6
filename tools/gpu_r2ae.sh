# LayerNorm forward rings: tests, micro-timings, XL step A/B; offload regression (lag default off)
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest -q --timeout 600 -p no:cacheprovider -rf tests/test_gpu_kernels.py tests/test_gpu_shapes.py \
   tests/test_gpu_offload.py tests/test_gpu_block.py > gpurun_out/pytest_ae.log 2>&1
echo "tests rc=$?"; grep -E "^(FAILED|ERROR)|^E  |passed|failed" gpurun_out/pytest_ae.log | head -20
for cfg in xl large; do for v in 1 0; do
  echo "== $cfg ring=$v"; NNT_LN_FWD_RING=$v timeout -s KILL 300 python tools/mem_bench.py --config $cfg --only ln_fwd 2>&1 | tail -1
done; done
for r in 1 2; do for v in 1 0; do
  NNT_LN_FWD_RING=$v timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_ae$v$r.log 2>&1
  echo "xl ring=$v"; python tools/summarize.py gpurun_out/bench_xl_ae$v$r.log | grep -E "value|ln_fwd"
done; done
