cd $GRAFT_REPO_ROOT
ONLY=${ONLY:-qkv,scores,scores+stats,dp_dA,out,fc+gelu,proj,proj_dx+gelu\',square8192}
for i in 1 2; do
for L in "" $ABLIBS; do
  echo "== lib: ${L:-working tree}"
  NNT_LIB=$L timeout 300 python tools/gemm_bench.py --only "$ONLY" 2>&1 | grep -v "^gemm\|total"
done
done
