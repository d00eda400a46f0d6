# GPT-2 small: 192-wide CTA-pair tiles for the N = 768 GEMMs (96 tiles of 256 x 256 on 74 pairs = 65 % of
# two rounds) -- tile choices and times with / without NNT_GEMM_192, then interleaved small and XL steps
cd $GRAFT_REPO_ROOT
NNT_DEBUG_GEMM=1 timeout -s KILL 300 python tools/gemm_bench.py --config small > gpurun_out/gs_def.log 2> gpurun_out/gs_def.err
NNT_GEMM_192=1 NNT_DEBUG_GEMM=1 timeout -s KILL 300 python tools/gemm_bench.py --config small > gpurun_out/gs_192.log 2> gpurun_out/gs_192.err
paste <(awk '{print $1, $(NF-1)}' gpurun_out/gs_def.log) <(awk '{print $(NF-1)}' gpurun_out/gs_192.log) | head -32
grep 'launch' gpurun_out/gs_192.err | sort | uniq -c | grep -E 'x768x|BN 192' | head -20
for i in 1 2 3; do
  python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab.log 2>/dev/null
  echo "small default: $(python tools/summarize.py gpurun_out/ab.log | head -1 | cut -c1-60)"
  NNT_GEMM_192=1 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab.log 2>/dev/null
  echo "small 192:     $(python tools/summarize.py gpurun_out/ab.log | head -1 | cut -c1-60)"
done
for i in 1 2; do
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>/dev/null
  echo "xl default: $(python tools/summarize.py gpurun_out/ab.log | head -1 | cut -c1-60)"
  NNT_GEMM_192=1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>/dev/null
  echo "xl 192:     $(python tools/summarize.py gpurun_out/ab.log | head -1 | cut -c1-60)"
done
