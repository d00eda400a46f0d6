cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_gpt2.py -q --timeout 200 -p no:cacheprovider 2>&1 | tail -3
timeout 120 python tools/ce_bench.py; NNT_CE_RESTREAM=1 timeout 120 python tools/ce_bench.py
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_ce.log 2>&1; python tools/summarize.py gpurun_out/bench_ce.log
