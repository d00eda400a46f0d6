# interleaved whole-step A/B of an env switch ($AB_ENV = 0 / 1), $AB_N rounds, same box
cd $GRAFT_REPO_ROOT
for i in $(seq 1 ${AB_N:-4}); do
for v in ${AB_VALS:-0 1}; do
  env $AB_ENV=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ab.log 2>/dev/null
  echo "$AB_ENV=$v: $(python tools/summarize.py gpurun_out/ab.log | head -1 | cut -c1-60)"
done
done
