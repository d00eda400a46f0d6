# compute-sanitizer over the small kernels' tests; capacity run (f4): XL width, 140 layers (> the
# 122 that fit resident), activations of 40 layers in pinned host memory
cd $GRAFT_REPO_ROOT
free -g | head -2
timeout -s KILL 1500 python bench.py --layers 140 --act-offload 40 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xl_L140_act40.log 2>&1
echo "L140 rc=$?"; tail -c 400 gpurun_out/bench_xl_L140_act40.log; python tools/summarize.py gpurun_out/bench_xl_L140_act40.log | head -1
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --act-offload 24 --no-cpu-baseline > gpurun_out/bench_xl_act24.log 2>&1
python tools/summarize.py gpurun_out/bench_xl_act24.log | head -1
bash tools/gpu_sanitize.sh > gpurun_out/sanitize_t.log 2>&1; cat gpurun_out/sanitize_t.log
