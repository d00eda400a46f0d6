cd $GRAFT_REPO_ROOT
for L in "" abtest/lnf3/libnnt.so abtest/lnf4/libnnt.so; do
NNT_LIB=$L python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.log 2>/dev/null
echo "lib=$L"; python tools/summarize.py gpurun_out/b.log | grep -E "value|ln_fwd"
done
