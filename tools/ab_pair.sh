# CTA-pair (cta_group::2) vs single-CTA tiles on the same box: GEMM tests, then gemm_bench
# alternating NNT_GEMM_CG=1 (single) and the default (pairs), then one bench.py per mode.
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_gemm.py -q --timeout 120 -p no:cacheprovider -x 2>&1 | tail -4
ONLY=${ONLY:-qkv,out,fc+gelu,proj,proj_dw,proj_dx+gelu\',fc_dw,fc_dx,out_dw,out_dx,qkv_dw,qkv_dx,square8192}
for i in 1 2; do
for CG in 1 0; do
  echo "== NNT_GEMM_CG=$CG"
  NNT_GEMM_CG=$CG timeout 300 python tools/gemm_bench.py --only "$ONLY" 2>&1 | grep -v "^gemm"
done
done
if [ -n "$BENCH" ]; then
  timeout 600 python -m pytest tests/test_gpu_block.py -q --timeout 180 -p no:cacheprovider -x 2>&1 | tail -3
  for CG in 1 0; do
    NNT_GEMM_CG=$CG timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cg$CG.log 2>&1
    python tools/summarize.py gpurun_out/bench_cg$CG.log | head -3
  done
fi
