# compute-sanitizer over the round-2 kernels: fused attention (stats / forward / new backward),
# LayerNorm-backward rings, embedding key sort, fused tensor-parallel SUM, stream-K GEMM
cd $GRAFT_REPO_ROOT
T="tests/test_gpu_attention.py tests/test_gpu_kernels.py::test_layernorm_bwd_ring_equals_group_kernel \
   tests/test_gpu_gpt2.py::test_embedding_bwd_bucket_order tests/test_gpu_tp.py::test_tp_fused_reduction_equals_summed_partials \
   tests/test_gpu_gemm.py::test_gemm_stream_k_bit_exact"
for tool in memcheck synccheck racecheck; do
  echo "== $tool"
  timeout -s KILL 1500 compute-sanitizer --tool $tool --print-limit 10 python -m pytest -q -p no:cacheprovider \
    --timeout 1400 -k "not 16384 and not 1024-4" $T > gpurun_out/san_$tool.log 2>&1
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Error:|Race reported" gpurun_out/san_$tool.log | sort | uniq -c | head -12
done
