cd $GRAFT_REPO_ROOT
for v in "0 " "1 " "1 abtest/pdlwait/libnnt.so" "0 "; do set -- $v
NNT_PDL=$1 NNT_LIB=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_v.log 2>&1
echo "PDL=$1 lib=$2"; python tools/summarize.py gpurun_out/bench_v.log 2>/dev/null | head -1
done
