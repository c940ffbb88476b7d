cd $GRAFT_REPO_ROOT
O=gpurun_out/r03l
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -k "relaxed_arithmetic" -q -p no:cacheprovider > $O/relaxed.log 2>&1; echo "rc=$?" >> $O/relaxed.log
NMODL_OPT_cdp5ish=lu_approx=1 NMODL_OPT_na6=lu_approx=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -k kinetic -q -p no:cacheprovider > $O/fullsize.log 2>&1; echo "rc=$?" >> $O/fullsize.log
for n in 1000000 10000000; do
  TUNE_N=$n timeout 600 python tools/tune.py --around "lu_approx=0,1" na6 cdp5ish >> $O/tune.jsonl 2>> $O/tune.err
done
for i in 1 2; do
NMODL_OPT_cdp5ish=lu_approx=1 NMODL_OPT_na6=lu_approx=1 timeout 600 python bench.py --no-cpu --no-e2e --no-sustained > $O/bench_lu1_$i.json 2> $O/bench_lu1_$i.err
timeout 600 python bench.py --no-cpu --no-e2e --no-sustained > $O/bench_lu0_$i.json 2> $O/bench_lu0_$i.err
done
