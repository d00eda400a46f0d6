# stream-K GEMM schedule: new + existing GEMM tests, per-GEMM timings (xl, small) with and without, step A/B
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest -q --timeout 600 -p no:cacheprovider -rf tests/test_gpu_gemm.py > gpurun_out/pytest_o_gemm.log 2>&1
echo "gemm tests rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_o_gemm.log | tail -15
for cfg in xl small; do
  timeout -s KILL 300 python tools/gemm_bench.py --config $cfg --iters 20 > gpurun_out/gemm_bench_${cfg}_sk.txt 2>&1
  NNT_GEMM_SK=0 timeout -s KILL 300 python tools/gemm_bench.py --config $cfg --iters 20 > gpurun_out/gemm_bench_${cfg}_nosk.txt 2>&1
  paste gpurun_out/gemm_bench_${cfg}_nosk.txt gpurun_out/gemm_bench_${cfg}_sk.txt | awk '{printf "%-14s %8s %8s | %8s %8s\n", $1, $6, $7, $13, $14}'
done
timeout -s KILL 1200 python -m pytest -q --timeout 900 -p no:cacheprovider -rf tests/test_gpu_block.py tests/test_gpu_gpt2.py tests/test_gpu_parity_full.py > gpurun_out/pytest_o_model.log 2>&1
echo "model tests rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_o_model.log | tail -15
for v in 1 0 1 0; do
  NNT_GEMM_SK=$v timeout -s KILL 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small_sk$v.log 2>&1
  echo "small sk=$v"; python tools/summarize.py gpurun_out/bench_small_sk$v.log | head -2
done
for v in 1 0; do
  NNT_GEMM_SK=$v timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_sk$v.log 2>&1
  echo "xl sk=$v"; python tools/summarize.py gpurun_out/bench_xl_sk$v.log | head -2
done
