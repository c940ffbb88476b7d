cd $GRAFT_REPO_ROOT
O=gpurun_out/r03q
mkdir -p $O
timeout 600 python tools/r03/na6_lu_parity.py > $O/parity.jsonl 2> $O/parity.err
for la in 2 3; do
NMODL_OPT_na6=lu_approx=$la timeout 900 python -m pytest tests/test_gpu_fullsize.py -k kinetic -q -p no:cacheprovider > $O/fullsize_$la.log 2>&1; echo "rc=$?" >> $O/fullsize_$la.log
done
for n in 1000000 10000000; do
  TUNE_N=$n timeout 600 python tools/tune.py --around "lu_approx=0,2,3" na6 >> $O/tune.jsonl 2>> $O/tune.err
done
