# out-projection tile choice with the TMA-staged residual: single-CTA 192 (default) vs CTA-pair 256 / 128
cd $GRAFT_REPO_ROOT
for i in 1 2; do
for cfg in xl small; do
  timeout -s KILL 300 python tools/gemm_bench.py --config $cfg --only out > gpurun_out/o1.log 2>&1; echo "$cfg default: $(tail -2 gpurun_out/o1.log | head -1)"
  NNT_GEMM_CG=2 NNT_GEMM_BN=256 timeout -s KILL 300 python tools/gemm_bench.py --config $cfg --only out > gpurun_out/o2.log 2>&1; echo "$cfg pair256: $(tail -2 gpurun_out/o2.log | head -1)"
  NNT_GEMM_CG=2 NNT_GEMM_BN=128 timeout -s KILL 300 python tools/gemm_bench.py --config $cfg --only out > gpurun_out/o3.log 2>&1; echo "$cfg pair128: $(tail -2 gpurun_out/o3.log | head -1)"
done
done
