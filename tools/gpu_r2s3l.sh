# attention task order: forward / statistics level groups (NNT_ATTN_FGROUP) and backward groups of 8
cd $GRAFT_REPO_ROOT
for g in 2 8; do
  NNT_ATTN_FGROUP=$g NNT_ATTN_BGROUP=$g timeout -s KILL 600 python -m pytest -q --timeout 600 -p no:cacheprovider tests/test_gpu_attention.py \
    tests/test_gpu_block.py -k "attn or attention or bf16" > gpurun_out/pytest_fg$g.log 2>&1; echo "GROUP=$g tests rc=$?"; tail -1 gpurun_out/pytest_fg$g.log
done
for g in 1 2 4 8; do
  NNT_ATTN_FGROUP=$g NNT_ATTN_BGROUP=$g timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:attn_ -c 8 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_fg$g.csv 2>/dev/null
  echo "== GROUP=$g"; grep -E 'attn_(stats|fwd_pv|bwd_kv)' gpurun_out/ncu_fg$g.csv | awk -F'","' '{split($0,a,"\""); print $5, $(NF-2), $NF}' | cut -c1-160 | tail -12
done
AB_ENV=NNT_ATTN_FGROUP AB_VALS="1 2 4 8" AB_N=3 BENCH_ARGS="" bash tools/ab_env_bench.sh
for i in 1 2 3; do for g in 4 8; do
  NNT_ATTN_BGROUP=$g python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab.log 2>/dev/null
  echo "BGROUP=$g: $(python tools/summarize.py gpurun_out/ab.log | head -1 | cut -c1-60)"
done; done
