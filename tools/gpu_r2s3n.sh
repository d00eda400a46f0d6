# LM-head GEMMs (XL and small widths) on the current path, blocked maps on / off
cd $GRAFT_REPO_ROOT
for b in 1 0; do
  echo "== BLOCKED=$b"
  NNT_GEMM_BLOCKED=$b NNT_DEBUG_GEMM=1 timeout -s KILL 300 python tools/lmhead_bench.py 1600 2> gpurun_out/lm_err$b.txt
  grep launch gpurun_out/lm_err$b.txt | sort | uniq -c
  NNT_GEMM_BLOCKED=$b timeout -s KILL 300 python tools/lmhead_bench.py 768
done
