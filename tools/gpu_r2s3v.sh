# attention backward level groups of 4 (NNT_ATTN_BGROUP) re-checked at HEAD, 4 interleaved XL pairs
cd $GRAFT_REPO_ROOT
AB_ENV=NNT_ATTN_BGROUP AB_VALS="1 4" AB_N=4 bash tools/ab_env_bench.sh
