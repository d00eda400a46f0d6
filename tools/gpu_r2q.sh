# stream-K (restricted) tests + interleaved XL step A/B; ncu --set full of the XL attention / LN / bias kernels
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest -q --timeout 600 -p no:cacheprovider -rf tests/test_gpu_gemm.py > gpurun_out/pytest_q_gemm.log 2>&1
echo "gemm tests rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_q_gemm.log | tail -8
for v in 1 0 1 0; do
  NNT_GEMM_SK=$v timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_q$v.log 2>&1
  echo "xl sk=$v"; python tools/summarize.py gpurun_out/bench_xl_q$v.log | head -2
done
for K in attn_fwd_pv_kernel attn_bwd_kv_kernel "gemm_tc_kernel<128, float, 3" ln_bwd "ln_fwd" colsum_partial adam_kernel; do
  tag=$(echo "$K" | tr -cd 'a-z_0-9')
  timeout -s KILL 600 ncu --profile-from-start off --set full --import-source on --clock-control none \
     --kernel-name-base demangled -k "regex:$K" -s 2 -c 1 -o gpurun_out/prof_xl_$tag -f \
     python tools/profile_step.py --config xl > gpurun_out/ncu_xl_$tag.log 2>&1
  tail -1 gpurun_out/ncu_xl_$tag.log
done
