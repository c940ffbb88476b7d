cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ag
mkdir -p $O
ncu --set full --import-source on --clock-control none -k regex:ProbAMPANMDA_EMS_k_step_nodes --launch-skip 3 --launch-count 1 -f -o $O/syn python tools/profile_bench.py --child synapse10m $O/meta.json > $O/ncu.log 2>&1
ncu -i $O/syn.ncu-rep --page source --csv --print-units base > $O/syn_source.csv 2> $O/src.err
ncu -i $O/syn.ncu-rep --page details --csv --print-units base > $O/syn_details.csv 2>> $O/src.err
rm -f $O/syn.ncu-rep
ls -la $O
