# A/B of whole training steps: the working tree's libnnt vs $ABLIBS (same box, interleaved)
cd $GRAFT_REPO_ROOT
for i in 1 2; do
for L in "" $ABLIBS; do
  NNT_LIB=$L python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ab.log 2>/dev/null
  echo "lib=${L:-working tree}: $(python tools/summarize.py gpurun_out/ab.log | head -1 | cut -c1-60)"
done
done
