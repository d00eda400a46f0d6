# interleaved XL step A/B: out-projection pair-256 rule (NNT_GEMM_OUT_PAIR) and the staged residual (NNT_GEMM_RES_SMEM)
cd $GRAFT_REPO_ROOT
AB_ENV=NNT_GEMM_OUT_PAIR AB_N=3 bash tools/ab_env_bench.sh
AB_ENV=NNT_GEMM_RES_SMEM AB_N=2 bash tools/ab_env_bench.sh
