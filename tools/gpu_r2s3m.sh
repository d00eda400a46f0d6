# compute-sanitizer over the session-3 kernel paths: narrow tail tiles, blocked 5-D MN-major maps (GEMM
# unit tests at reduced shapes), the ZeRO-1 bf16 shadow gather at world 1 (NCCL) and the GPT-2 small block
cd $GRAFT_REPO_ROOT
T="tests/test_gpu_gemm.py::test_gemm_blocked_mn_major_maps_bit_exact tests/test_gpu_gemm.py::test_gemm_cta_pair_bit_exact \
   tests/test_gpu_gemm.py::test_gemm_narrow_tail_bit_exact tests/test_gpu_dp.py::test_zero1_world1_equals_single_gpu_bitwise"
for tool in memcheck synccheck; do
  echo "== $tool"
  timeout -s KILL 1500 compute-sanitizer --tool $tool --print-limit 10 python -m pytest -q -p no:cacheprovider \
    --timeout 1400 -k "not 8192x1600x1600 and not 1600x1600x8192" $T 2>&1 | tail -6
done
