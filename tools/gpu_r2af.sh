# M-outer tile raster for tall GEMMs: tests, per-GEMM XL / small timings, DRAM bytes, step A/B
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest -q --timeout 600 -p no:cacheprovider -rf tests/test_gpu_gemm.py tests/test_gpu_block.py > gpurun_out/pytest_af.log 2>&1
echo "tests rc=$?"; grep -E "^(FAILED|ERROR)|^E  |passed|failed" gpurun_out/pytest_af.log | head -10
G="qkv,out,fc+gelu,proj_plain,proj,proj_dw,proj_dx+gelu',fc_dw,fc_dx,out_dw,out_dx,qkv_dw,qkv_dx"
for cfg in xl small; do
  NNT_GEMM_ORDER=1 timeout -s KILL 300 python tools/gemm_bench.py --config $cfg --iters 20 --no-ws --only "$G" > gpurun_out/gb_o1.txt 2>&1
  NNT_GEMM_ORDER=0 timeout -s KILL 300 python tools/gemm_bench.py --config $cfg --iters 20 --no-ws --only "$G" > gpurun_out/gb_o0.txt 2>&1
  echo "== $cfg  (order0 | order1)"; paste gpurun_out/gb_o0.txt gpurun_out/gb_o1.txt | awk '{printf "%-14s %8s | %8s\n", $1, $6, $13}'
done
for v in 1 0; do
  NNT_GEMM_ORDER=$v timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
    -k regex:gemm_tc_kernel -s 3 -c 1 --log-file gpurun_out/ord$v.csv python tools/gemm_bench.py --config xl --only proj_plain --iters 1 --no-ws > /dev/null 2>&1
  echo "proj_plain order=$v"; grep -E "gpu__time|dram__bytes" gpurun_out/ord$v.csv | awk -F'","' '{print $(NF-2)" "$NF}'
done
for r in 1 2; do for v in 1 0; do
  NNT_GEMM_ORDER=$v timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_af$v$r.log 2>&1
  echo "xl order=$v"; python tools/summarize.py gpurun_out/bench_xl_af$v$r.log | head -2
done; done
for v in 1 0; do
  NNT_GEMM_ORDER=$v timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_af$v.log 2>&1
  echo "small order=$v"; python tools/summarize.py gpurun_out/bench_small_af$v.log | head -2
done
