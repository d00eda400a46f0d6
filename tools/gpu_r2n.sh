# XL analysis: per-GEMM times vs cuBLAS, one-step launch list + per-class DRAM traffic (xl, small),
# one ncu --set full capture of the XL FC+GELU and proj GEMMs
cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python tools/gemm_bench.py --config xl --iters 20 > gpurun_out/gemm_bench_xl.txt 2>&1; cat gpurun_out/gemm_bench_xl.txt
timeout -s KILL 300 python tools/cublas_bench.py 1600 > gpurun_out/cublas_1600.txt 2>&1; cat gpurun_out/cublas_1600.txt
for cfg in xl small; do
timeout -s KILL 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none --csv --log-file gpurun_out/traffic_$cfg.csv python tools/profile_step.py --config $cfg --trace gpurun_out/trace_$cfg.json \
   > gpurun_out/ncu_traffic_$cfg.log 2>&1
python tools/traffic.py gpurun_out/traffic_$cfg.csv gpurun_out/trace_$cfg.json gpurun_out/traffic_$cfg.json
done
for ONLY in fc+gelu proj; do
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 3 -c 1 -o gpurun_out/prof_xl_$ONLY -f python tools/gemm_bench.py --config xl --only $ONLY --iters 1 > gpurun_out/ncu_gemm_$ONLY.log 2>&1
tail -1 gpurun_out/ncu_gemm_$ONLY.log
done
