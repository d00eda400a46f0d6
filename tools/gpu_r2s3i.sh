# round-2 session-3 checkpoint: full GPU suite, smoke, bench XL + small, torchrun N=1, XL one-step launch list
cd $GRAFT_REPO_ROOT
export NNT_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_s3i.jsonl
rm -f $NNT_PARITY_LOG
timeout -s KILL 2400 python -m pytest tests -m gpu -q --timeout 1800 -p no:cacheprovider -rf > gpurun_out/pytest_s3i.log 2>&1
echo "pytest rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_s3i.log | tail -25
unset NNT_PARITY_LOG
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke_s3i.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_s3i.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_xl_s3i.log 2>&1; echo "bench xl rc=$?"; python tools/summarize.py gpurun_out/bench_xl_s3i.log
timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_s3i.log 2>&1; python tools/summarize.py gpurun_out/bench_small_s3i.log
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun1_s3i.log 2>&1; echo "torchrun rc=$?"; tail -c 600 gpurun_out/bench_torchrun1_s3i.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_xl_s3i.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_xl_s3i.log 2>&1; echo "ncu rc=$?"
python tools/summarize.py gpurun_out/launches_xl_s3i.csv | head -30
