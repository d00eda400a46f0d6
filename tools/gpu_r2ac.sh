# value of the backward's side stream: interleaved XL / small steps with NNT_SIDE_STREAM=1 / 0
cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in 1 0; do
  NNT_SIDE_STREAM=$v timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_ac$v$r.log 2>&1
  echo "xl side=$v"; python tools/summarize.py gpurun_out/bench_xl_ac$v$r.log | head -1
  NNT_SIDE_STREAM=$v timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_ac$v$r.log 2>&1
  echo "small side=$v"; python tools/summarize.py gpurun_out/bench_small_ac$v$r.log | head -1
done; done
