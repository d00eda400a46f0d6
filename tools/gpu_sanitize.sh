# compute-sanitizer memcheck / synccheck / initcheck (and racecheck on the smaller kernels) over
# the tiny fp32 block, the bf16 block at S = 256 (fused attention, tcgen05 GEMMs, LayerNorm,
# softmax passes, Adam), the GEMM unit tests, the fused attention kernels and the world-1 DP path.
cd $GRAFT_REPO_ROOT
T="tests/test_gpu_block.py::test_tiny_fp32_fwd_bwd_adam tests/test_gpu_block.py::test_bf16_gpt2_small_block \
   tests/test_gpu_attention.py tests/test_gpu_gemm.py::test_gemm_cta_pair_bit_exact \
   tests/test_gpu_gemm.py::test_gemm_split_k_shared_workspace_shapes tests/test_gpu_kernels.py::test_layernorm_bwd \
   tests/test_gpu_dp.py::test_dp_path_world1_equals_single_gpu_bitwise"
for tool in memcheck synccheck initcheck; do
  echo "== $tool"
  timeout -s KILL 1500 compute-sanitizer --tool $tool --print-limit 10 python -m pytest -q -p no:cacheprovider \
    --timeout 1400 -k "not 1024" $T 2>&1 | tail -6
done
echo "== racecheck (shared-memory hazards; LayerNorm / column merges / GEMM tests)"
timeout -s KILL 1500 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest -q -p no:cacheprovider \
  --timeout 1400 tests/test_gpu_kernels.py::test_layernorm_bwd tests/test_gpu_kernels.py::test_bias_grad \
  "tests/test_gpu_gemm.py::test_gemm_cta_pair_bit_exact" tests/test_gpu_attention.py 2>&1 | tail -6
