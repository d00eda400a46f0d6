# compute-sanitizer memcheck / racecheck / synccheck over the kernels added late in the round
cd $GRAFT_REPO_ROOT
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --print-limit 5 python -m pytest -q -p no:cacheprovider \
    "tests/test_gpu_gpt2.py::test_cross_entropy_kernel" "tests/test_gpu_gemm.py::test_attn_rowdot_head_dims" 2>&1 | tail -4
done
