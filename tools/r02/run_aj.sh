cd $GRAFT_REPO_ROOT
O=gpurun_out/r02aj
mkdir -p $O/prof
cp profiles/ncu_traffic.json $O/prof/ncu_traffic.json
PROFILE_TAG=r02fin_prof timeout 1500 python tools/profile_bench.py $O/prof bbp20m bbp20m_grouped column > $O/profile.log 2>&1; echo "rc=$?" >> $O/profile.log
rm -f $O/prof/*.ncu-rep
cp $O/prof/ncu_traffic.json profiles/ncu_traffic.json
timeout 600 python bench.py --workload bbp20m_grouped --no-also --no-e2e --no-cpu > $O/bbpg.json 2> $O/bbpg.err
timeout 600 python bench.py --workload bbp20m --no-also --no-e2e --no-cpu > $O/bbp.json 2> $O/bbp.err
timeout 600 python bench.py --workload column > $O/col.json 2> $O/col.err
timeout 600 python bench.py --workload column --cells 12500 --no-e2e --no-cpu > $O/col12.json 2> $O/col12.err
timeout 900 python -m pytest tests/test_gpu_column.py tests/test_gpu_fullsize.py -q -p no:cacheprovider > $O/gputests.log 2>&1; echo "rc=$?" >> $O/gputests.log
