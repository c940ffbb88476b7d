cd $GRAFT_REPO_ROOT
O=gpurun_out/r03n
mkdir -p $O
PROFILE_TAG=r03fin_prof timeout 1500 python tools/profile_bench.py $O/prof kinetic1m kinetic10m kinetic1m_grouped > $O/profile.log 2>&1; echo "rc=$?" >> $O/profile.log
rm -f $O/prof/*.ncu-rep
