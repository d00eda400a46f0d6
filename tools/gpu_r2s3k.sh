# XL bench-shape block parity (every gradient + Adam); attention backward level groups (NNT_ATTN_BGROUP) A/B
cd $GRAFT_REPO_ROOT
export NNT_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_s3k.jsonl
rm -f $NNT_PARITY_LOG
timeout -s KILL 1500 python -m pytest -q --timeout 1500 -p no:cacheprovider -rf --durations=3 \
  tests/test_gpu_shapes.py::test_xl_bench_shape_block_every_gradient > gpurun_out/pytest_s3k.log 2>&1
echo "rc=$?"; grep -E "passed|failed|^E |call " gpurun_out/pytest_s3k.log | head -20
python tools/parity_summary.py gpurun_out/parity_s3k.jsonl 2>&1 | head -40
unset NNT_PARITY_LOG
for g in 2 4; do
  NNT_ATTN_BGROUP=$g timeout -s KILL 600 python -m pytest -q --timeout 600 -p no:cacheprovider tests/test_gpu_attention.py \
    tests/test_gpu_block.py -k "attn or attention or bf16" > gpurun_out/pytest_bg$g.log 2>&1; echo "BGROUP=$g tests rc=$?"; tail -1 gpurun_out/pytest_bg$g.log
done
for g in 1 2 4; do
  NNT_ATTN_BGROUP=$g timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none \
    -k regex:attn_bwd_kv -c 4 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bg$g.csv 2>/dev/null
  echo "== BGROUP=$g"; grep attn_bwd gpurun_out/ncu_bg$g.csv | awk -F'","' '{print $(NF-2), $NF}' | tail -4
done
AB_ENV=NNT_ATTN_BGROUP AB_VALS="1 2 4" AB_N=3 bash tools/ab_env_bench.sh
