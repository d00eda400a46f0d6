# bench lines for every BASELINE config that fits one GPU (full GPT-2 large / XL, the wide block)
cd $GRAFT_REPO_ROOT
for c in large xl wide; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  grep '^{' gpurun_out/bench_$c.log | tail -1 > gpurun_out/bench_$c.json
  python tools/summarize.py gpurun_out/bench_$c.log | head -3
done
