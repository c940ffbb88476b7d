cd $GRAFT_REPO_ROOT
O=gpurun_out/r03f
mkdir -p $O
for n in 1100000 1150000 1212416 1230000 1250000 1300000 1400000 1818000; do
  nodes=$((n * 21 / 100))
  TUNE_N=$n TUNE_NODES=$nodes timeout 300 python tools/tune.py --around "pipe=0" ProbAMPANMDA_EMS >> $O/syn_sizes.jsonl 2>> $O/syn_sizes.err
done
