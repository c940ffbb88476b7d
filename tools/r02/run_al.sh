cd $GRAFT_REPO_ROOT
O=gpurun_out/r02al
mkdir -p $O/prof
cp profiles/ncu_traffic.json $O/prof/ncu_traffic.json
PROFILE_TAG=r02fin_prof timeout 900 python tools/profile_bench.py $O/prof bbp20m_grouped > $O/profile.log 2>&1; echo "rc=$?" >> $O/profile.log
rm -f $O/prof/*.ncu-rep
