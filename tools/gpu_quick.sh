# quick GPU loop: targeted tests + HBM kernel micro-timings + one bench line
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_gpt2.py tests/test_gpu_block.py -q --timeout 200 -p no:cacheprovider 2>&1 | tail -3
timeout 200 python tools/mem_bench.py 2>&1 | tail -20
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_q.log 2>&1; python tools/summarize.py gpurun_out/bench_q.log
