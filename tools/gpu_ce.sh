cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_gpt2.py -q --timeout 200 -p no:cacheprovider 2>&1 | tail -3
timeout 120 python tools/ce_bench.py; NNT_CE_RESTREAM=1 timeout 120 python tools/ce_bench.py
