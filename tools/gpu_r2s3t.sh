# out-projection with CTA pairs at the tile model's width (NNT_GEMM_CG=2, no BN forcing)
cd $GRAFT_REPO_ROOT
for i in 1 2; do
for cfg in xl small; do
  timeout -s KILL 300 python tools/gemm_bench.py --config $cfg --only out > gpurun_out/o1.log 2>&1; echo "$cfg default: $(tail -2 gpurun_out/o1.log | head -1)"
  NNT_DEBUG_GEMM=1 NNT_GEMM_CG=2 timeout -s KILL 300 python tools/gemm_bench.py --config $cfg --only out > gpurun_out/o2.log 2>gpurun_out/o2.err; echo "$cfg pair: $(tail -2 gpurun_out/o2.log | head -1)"; grep launch gpurun_out/o2.err | sort | uniq -c
done
done
