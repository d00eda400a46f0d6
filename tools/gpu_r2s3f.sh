# attention backward: blocked P map (one TMA request per 128x128 P tile), tests + step A/B
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest -q --timeout 600 -p no:cacheprovider -rf tests/test_gpu_attention.py \
  tests/test_gpu_block.py > gpurun_out/pytest_s3f.log 2>&1
echo "tests rc=$?"; grep -E "^(FAILED|ERROR)|^E  |passed|failed" gpurun_out/pytest_s3f.log | head -20
for v in 0 1; do
  NNT_ATTN_PBLK=$v timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none \
    -k regex:attn_bwd_kv -c 6 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_pblk$v.csv 2>/dev/null
  echo "== PBLK=$v"; grep attn_bwd gpurun_out/ncu_pblk$v.csv | awk -F'","' '{print $(NF-2), $NF}' | tail -6
done
AB_ENV=NNT_ATTN_PBLK AB_N=3 bash tools/ab_env_bench.sh
